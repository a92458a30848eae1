"""Generic step kernel with its side records computed ahead by side_kernel
(CLAW_SIDE=1) or inside the step kernel (CLAW_SIDE=0): the same helpers in the
same order, so the results must be bitwise equal -- on ragged levels for every
limiter and transverse order, several tile heights, and the C3 hierarchy."""
import numpy as np
import pytest

from paper_1808_02638_b200 import binding, workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    binding.load()


def run_level(descs, q0, side, limiter, ot, tile_rows, bc, steps, monkeypatch):
    monkeypatch.setenv("CLAW_SIDE", "1" if side else "0")
    monkeypatch.setenv("CLAW_LANE", "0")  # the side-pass kernel (not the halo-lane one)
    g = binding.Claw(W.DOMAIN, bc, limiter, ot, device=0, tile_rows=tile_rows, path=1)
    g.set_level(1, descs, q0)
    dt = (0.8 if ot else 0.4) * 2.0 / 40
    c = [0.0]
    for n in range(steps):
        g.fill_ghost(1, n * dt)
        c.append(g.advance_level(1, dt))
    st = g.stats()
    out = g.read_level(1)
    g.close()
    return out, c, st


@pytest.mark.parametrize("limiter,ot,tile_rows,bc", [(4, 2, 0, W.EXTRAP), (3, 2, 16, W.PERIODIC), (1, 1, 7, W.EXTRAP),
                                                     (0, 0, 64, W.PERIODIC), (2, 2, 32, (1, 1, 2, 2))])
def test_side_kernel_bitwise_equals_in_kernel_side_passes(limiter, ot, tile_rows, bc, monkeypatch):
    descs = W.ragged_level(11 + limiter, nx=40, ny=36, max_w=13)
    q0 = W.random_ic(descs, 5 + limiter)
    a, ca, sa = run_level(descs, q0, True, limiter, ot, tile_rows, bc, 5, monkeypatch)
    b, cb, sb = run_level(descs, q0, False, limiter, ot, tile_rows, bc, 5, monkeypatch)
    assert np.array_equal(a, b) and ca == cb
    assert sa["ghost_launches"] == sb["ghost_launches"] + 5     # one side_kernel per step


def test_side_kernel_on_c3_hierarchy(monkeypatch):
    wl = W.c3()
    q0s = W.hierarchy_ic(wl)
    res = []
    for side in (True, False):
        monkeypatch.setenv("CLAW_SIDE", "1" if side else "0")
        monkeypatch.setenv("CLAW_LANE", "0")  # the side-pass kernel (not the halo-lane one)
        g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0)
        for L, (lv, q) in enumerate(zip(wl.levels, q0s), start=1):
            g.set_level(L, lv.descs, q)
        dt = wl.dt0()
        cfl = [g.advance_hierarchy(n * dt, dt, update=True) for n in range(2)]
        res.append(([g.read_level(L) for L in (1, 2, 3)], cfl))
        g.close()
    assert res[0][1] == res[1][1]
    for x, y in zip(res[0][0], res[1][0]):
        assert np.array_equal(x, y)
