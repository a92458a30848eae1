"""The halo-lane generic kernel (`step_lane_kernel`, default for
generic levels) against the side-pass generic kernel (CLAW_LANE=0): the same
cell arithmetic on the same ghost sources, so results must agree bit for bit.
Cases: ragged levels (widths 1..40, T-junction neighbours, every limiter and
order_trans, both BCs, non-uniform media), multi-level hierarchies with
coarse-interpolated ghosts (C2, C3 forced generic), the conservation fix,
Morton-partitioned virtual ranks (remote frame ghosts), and the oracle."""
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


def run_level(d, q0, bc, limiter, ot, nsteps, dt, lane, monkeypatch, tile_rows=0):
    monkeypatch.setenv("CLAW_LANE", "1" if lane else "0")
    g = binding.Claw(W.DOMAIN, bc, limiter, ot, device=0, path=1, tile_rows=tile_rows)
    g.set_level(1, d, q0)
    assert g.level_mode(1) == "generic"
    cfl = []
    for n in range(nsteps):
        g.fill_ghost(1, n * dt)
        cfl.append(g.advance_level(1, dt))
    pc = [g.patch_cfl(1, p) for p in range(len(d))]
    out = g.read_level(1)
    g.close()
    return out, cfl, pc


@pytest.mark.parametrize("limiter", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("order_trans", [0, 1, 2])
@pytest.mark.parametrize("bc", [W.EXTRAP, W.PERIODIC, (1, 1, 2, 2)])
def test_lane_equals_side_pass_kernel_ragged(limiter, order_trans, bc, monkeypatch):
    d = W.ragged_level(3 + limiter, 75, 52, 40)
    q0 = W.random_ic(d, 10 * limiter + order_trans)
    dt = (0.9 if order_trans else 0.45) * float(d["dx"][0])
    a = run_level(d, q0, bc, limiter, order_trans, 6, dt, True, monkeypatch)
    b = run_level(d, q0, bc, limiter, order_trans, 6, dt, False, monkeypatch)
    assert np.array_equal(a[0], b[0]) and a[1] == b[1] and a[2] == b[2]


@pytest.mark.parametrize("tile_rows", [0, 7, 16, 64])
def test_lane_tile_rows_and_oracle(tile_rows, monkeypatch):
    """Tile heights (ragged last tiles, 4-phase overshoot) and 60 steps of the
    lane kernel against the oracle at the north_star bar."""
    d = W.ragged_level(21, 96, 80, 40)
    q0 = W.random_ic(d, 21)
    dt = 0.9 * float(d["dx"][0])
    a = run_level(d, q0, W.EXTRAP, 4, 2, 60, dt, True, monkeypatch, tile_rows=tile_rows)
    o = oracle.Oracle(W.DOMAIN, W.EXTRAP, 4, 2, nthreads=0)
    o.set_level(1, d, q0)
    for n in range(60):
        o.fill_ghost(1, n * dt)
        assert o.advance_level(1, dt) == a[1][n]
    qo = o.read_level(1)
    assert float(np.abs(a[0] - qo).max() / np.abs(qo).max()) <= TOL


def test_lane_non_uniform_media(monkeypatch):
    """Per-patch rho, K (R12): per-tile constants in the kernel."""
    d = W.ragged_level(8, 60, 44, 30)
    rng = np.random.default_rng(8)
    d["rho"] = rng.uniform(0.5, 2.0, len(d))
    d["K"] = rng.uniform(0.5, 2.0, len(d))
    q0 = W.random_ic(d, 8)
    dt = 0.4 * float(d["dx"][0])
    a = run_level(d, q0, W.EXTRAP, 4, 2, 5, dt, True, monkeypatch)
    b = run_level(d, q0, W.EXTRAP, 4, 2, 5, dt, False, monkeypatch)
    assert np.array_equal(a[0], b[0]) and a[1] == b[1] and a[2] == b[2]


@pytest.mark.parametrize("name,reflux", [("c2", False), ("c2", True), ("c3", False)])
def test_lane_hierarchy_bitwise(name, reflux, monkeypatch):
    """Coarse-interpolated frame ghosts, updating and (optionally) the
    conservation fix through Berger-Oliger cycles; every level generic."""
    wl = getattr(W, name)()
    levels = [lv.descs for lv in wl.levels]
    q0s = W.hierarchy_ic(wl)
    res = []
    for lane in (True, False):
        monkeypatch.setenv("CLAW_LANE", "1" if lane else "0")
        g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0, path=1, reflux=reflux)
        for L, (d, q) in enumerate(zip(levels, q0s), start=1):
            g.set_level(L, d, q)
        dt = 0.9 * float(levels[0]["dx"][0])
        cfl = [g.advance_hierarchy(n * dt, dt, update=True) for n in range(3)]
        res.append(([g.read_level(L) for L in range(1, len(levels) + 1)], cfl))
        g.close()
    assert res[0][1] == res[1][1]
    for x, y in zip(res[0][0], res[1][0]):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("world,bc", [(3, W.PERIODIC), (5, (1, 1, 2, 2))])
def test_lane_morton_virtual_ranks(world, bc, monkeypatch):
    """Morton-partitioned ragged level on virtual ranks (remote ghosts in the
    frame, interior tiles launched before edge tiles): bitwise equal to one
    rank."""
    monkeypatch.setenv("CLAW_LANE", "1")
    d = W.ragged_level(6, 90, 70, 30)
    q0 = W.random_ic(d, world)
    offs = W.level_offsets(d)
    owners = binding.partition(d, world)
    ctxs = []
    for r in range(world):
        c = binding.Claw(W.DOMAIN, bc, 4, 2, device=0, rank=r, world=world, exchange=1)
        c.set_level(1, d, np.concatenate([q0[offs[p]:offs[p + 1]] for p in range(len(d)) if owners[p] == r]))
        assert c.level_mode(1) == "generic"
        ctxs.append(c)
    ref = binding.Claw(W.DOMAIN, bc, 4, 2, device=0)
    ref.set_level(1, d, q0)
    dt = 0.9 * float(d["dx"][0])
    for n in range(4):
        for c in ctxs:
            c.fill_ghost(1, n * dt)
        for r in range(world):
            for s in range(world):
                if r != s:
                    ctxs[s].halo_unpack(1, r, ctxs[r].halo_pack(1, s))
        cfl = max(c.advance_level(1, dt) for c in ctxs)
        ref.fill_ghost(1, n * dt)
        assert cfl == ref.advance_level(1, dt)
    full = ref.read_level(1)
    for r, c in enumerate(ctxs):
        mine = np.concatenate([full[offs[p]:offs[p + 1]] for p in range(len(d)) if owners[p] == r])
        assert np.array_equal(c.read_level(1), mine)
    for c in ctxs + [ref]:
        c.close()
