"""Row copies of the grid and vc kernels ("Row copies"):
the 16-byte per-lane copies of interior strips (RC 1 with 4-warp CTAs, RC 2
with one-warp CTAs -- chosen by launch size where the layout allows them) and
the per-lane 8-byte copies (RC 0, CLAW_ROWCOPY=0) feed the same arithmetic,
so the results are bitwise equal; and all match the oracle.  The sparse
lattice (RC 2 vs RC 0) is covered at the end.  Shapes cover patch widths where a 34-column ring row spans 1, 2 or 3
patches (even widths 2 .. 130), levels just wider than one or two strips
(edge strips fall back to 8-byte copies), tiles spanning patch rows, and both
BCs.  CLAW_ROWCOPY is read when a context is created (one setting per
process at a time: each run finishes before the next context exists).
"""
import numpy as np
import pytest

import oracle
from paper_1808_02638_b200 import binding, workloads as W

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    binding.load()


def rel_err(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def run_grid(monkeypatch, rc, d, q0, bc, limiter, ot, dt, nsteps, aux=None, th=None):
    monkeypatch.setenv("CLAW_ROWCOPY", str(rc))
    if th:
        monkeypatch.setenv("CLAW_GRID_TH", str(th))
    g = binding.Claw(W.DOMAIN, bc, limiter, ot, device=0)
    g.set_level(1, d, q0)
    assert g.level_mode(1) == "grid"
    if aux is not None:
        g.set_aux(1, aux)
    cfl = []
    for n in range(nsteps):
        g.fill_ghost(1, n * dt)
        cfl.append(g.advance_level(1, dt))
    q = g.read_level(1)
    g.close()
    return q, cfl


def oracle_run(d, q0, bc, limiter, ot, dt, nsteps, aux=None):
    o = oracle.Oracle(W.DOMAIN, bc, limiter, ot, nthreads=0)
    o.set_level(1, d, q0)
    if aux is not None:
        o.set_aux(1, aux)
    for n in range(nsteps):
        o.fill_ghost(1, n * dt)
        o.advance_level(1, dt)
    return o.read_level(1)


# (npx, npy, mx, my): mx 2 / 18 / 34 -> 3+ / 2-3 / 2 patches per ring row;
# NX = 62, 64, 92 put the last strip's window at / past the level edge
# (3 mx my a multiple of 32: gapless 256-byte aligned patches, grid mode)
SHAPES = [(31, 2, 2, 16, W.EXTRAP, 4, 2), (4, 3, 18, 16, W.PERIODIC, 1, 2), (2, 2, 34, 16, W.EXTRAP, 2, 1),
          (2, 2, 32, 32, W.PERIODIC, 4, 0), (1, 3, 92, 8, (2, 2, 1, 1), 3, 2), (3, 2, 130, 16, W.EXTRAP, 4, 2),
          (8, 8, 64, 64, W.EXTRAP, 4, 2)]


@pytest.mark.parametrize("npx,npy,mx,my,bc,limiter,ot", SHAPES)
def test_grid_row_copies_bitwise(monkeypatch, npx, npy, mx, my, bc, limiter, ot):
    d = W.uniform_level(npx, npy, mx, my)
    q0 = W.random_ic(d, 13 * mx + my)
    dt = (0.9 if ot else 0.45) * 2 / max(npx * mx, npy * my)
    q0c, c0 = run_grid(monkeypatch, 0, d, q0, bc, limiter, ot, dt, 6)
    for rc in (1, 2):   # 16-byte copies with 4-warp / one-warp CTAs
        q1c, c1 = run_grid(monkeypatch, rc, d, q0, bc, limiter, ot, dt, 6)
        assert np.array_equal(q0c, q1c) and c0 == c1, rc
    assert rel_err(q1c, oracle_run(d, q0, bc, limiter, ot, dt, 6)) <= TOL


@pytest.mark.parametrize("th", [64, 96])
def test_grid_row_copies_spanning_tiles_bitwise(monkeypatch, th):
    d = W.uniform_level(5, 6, 32, 32)
    q0 = W.random_ic(d, th)
    dt = 0.9 * 2 / 192
    a = run_grid(monkeypatch, 0, d, q0, W.EXTRAP, 4, 2, dt, 5, th=th)
    for rc in (1, 2):
        b = run_grid(monkeypatch, rc, d, q0, W.EXTRAP, 4, 2, dt, 5, th=th)
        assert np.array_equal(a[0], b[0]) and a[1] == b[1], rc


@pytest.mark.parametrize("npx,npy,mx,my,bc", [(4, 3, 18, 16, W.PERIODIC), (2, 2, 34, 16, W.EXTRAP),
                                              (3, 2, 64, 24, W.EXTRAP), (31, 2, 2, 16, W.PERIODIC)])
def test_vc_row_copies_bitwise(monkeypatch, npx, npy, mx, my, bc):
    """step_vc_kernel: 16-byte copies of (p, u, v) from q and (Z, c) from aux
    vs per-lane 8-byte copies; random media."""
    d = W.uniform_level(npx, npy, mx, my)
    aux = W.random_media(d, mx + 3 * my)
    q0 = W.random_ic(d, mx + my)
    dt = 0.8 * min(float(d["dx"][0]), float(d["dy"][0])) / W.max_sound_speed(aux, d)
    a = run_grid(monkeypatch, 0, d, q0, bc, 4, 2, dt, 6, aux=aux)
    b = run_grid(monkeypatch, 1, d, q0, bc, 4, 2, dt, 6, aux=aux)
    assert np.array_equal(a[0], b[0]) and a[1] == b[1]
    assert rel_err(b[0], oracle_run(d, q0, bc, 4, 2, dt, 6, aux=aux)) <= TOL


def test_sparse_lattice_row_copies_bitwise(monkeypatch):
    """The sparse-lattice grid kernel (C3's level 3) with 16-byte copies
    (chunks from patch or virtual frame slots, one-warp CTAs) vs per-lane
    8-byte copies: whole-hierarchy runs bitwise equal.  (The ratio-2 / 4
    lattices of test_gpu_parity's sparse test run the default copies against
    the generic kernel.)"""
    wl = W.c3()
    res = []
    for rc in (0, 3):
        monkeypatch.setenv("CLAW_ROWCOPY", str(rc))
        g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0)
        for L, (lv, q) in enumerate(zip(wl.levels, W.hierarchy_ic(wl)), start=1):
            g.set_level(L, lv.descs, q)
        assert g.level_mode(3) == "sparse"
        dt = wl.dt0()
        cfl = [g.advance_hierarchy(n * dt, dt, update=True) for n in range(3)]
        res.append(([g.read_level(L) for L in range(1, 4)], cfl))
        g.close()
    assert all(np.array_equal(a, b) for a, b in zip(res[0][0], res[1][0])) and res[0][1] == res[1][1]
