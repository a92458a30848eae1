"""GPU parity at north_star length (BASELINE.json: max|q_gpu - q_oracle| <=
1e-12 max|q_oracle| "after 100 steps"; C2 runs 200 coarse
steps, C3 100).

* C2 for 200 and C3 for 100 coarse steps (1 + R1 + R1 R2 level advances each,
  P:113-118), as plain Berger-Oliger cycles, with updating and with
  updating plus the conservation fix (R17).  The GPU runs
  the native claw_advance_hierarchy (the bench's driver); the oracle runs the
  recursion level step by level step.
* The default bench workload (C5, 16384^2 cells, grid kernel with 256-row
  tiles spanning patch rows) and C4 at full size over several consecutive
  steps: every step, sampled 3x3 patch blocks are read from the GPU state and
  the oracle advances them one step; the GPU's next state must match.
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


def oracle_cycle(o, L, t, dt, nlev, ratios, update):
    """One Berger-Oliger step of level L with its R sub-steps of L+1
    (recursively), then (update) averaging + fix of L from L+1."""
    o.fill_ghost(L, t)
    c = o.advance_level(L, dt)
    if L < nlev:
        R = ratios[L - 1]
        for k in range(R):
            c = max(c, oracle_cycle(o, L + 1, t + k * dt / R, dt / R, nlev, ratios, update))
        if update:
            o.update_level(L + 1)
    return c


@pytest.mark.parametrize("mode", ["plain", "update", "reflux"])
@pytest.mark.parametrize("name,steps", [("c2", 200), ("c3", 100)])
def test_hierarchy_at_north_star_length(name, steps, mode):
    wl = getattr(W, name)()
    q0s = W.hierarchy_ic(wl)
    nlev = len(wl.levels)
    ratios = [wl.levels[L].ratio for L in range(1, nlev)]
    reflux = mode == "reflux"
    update = mode != "plain"
    g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0, reflux=reflux)
    o = oracle.Oracle(wl.domain, wl.bc, wl.limiter, wl.order_trans, nthreads=0, reflux=reflux)
    for L, (lv, q0) in enumerate(zip(wl.levels, q0s), start=1):
        g.set_level(L, lv.descs, q0)
        o.set_level(L, lv.descs, q0)
    dt = wl.dt0()
    for n in range(steps):
        cg = g.advance_hierarchy(n * dt, dt, update=update)
        co = oracle_cycle(o, 1, n * dt, dt, nlev, ratios, update)
        assert cg == co, (n, cg, co)
    errs = [rel_err(g.read_level(L), o.read_level(L)) for L in range(1, nlev + 1)]
    g.close()
    assert max(errs) <= TOL, errs


def sampled_steps(wl, m, nsteps, seed, samples_per_step):
    """nsteps consecutive full-size GPU steps; before each, sampled 3x3 patch
    blocks of the GPU state q^n are read, and the oracle's one step of them
    must equal the GPU's q^{n+1} on the centre patch."""
    d = wl.levels[0].descs
    npx = int(round(np.sqrt(len(d))))
    g = binding.Claw(W.DOMAIN, W.EXTRAP, 4, 2, device=0)
    g.set_level(1, d, W.random_ic(d, seed))
    assert g.level_mode(1) == "grid"
    dt = wl.dt0()
    dx = float(d["dx"][0])
    rng = np.random.default_rng(seed)
    edge = [(0, 0), (npx - 1, npx - 1), (0, npx - 1), (npx - 1, 0), (3, npx // 2), (npx // 2, npx - 1)]
    checked = 0
    for n in range(nsteps):
        samples = [tuple(x) for x in rng.integers(0, npx, (samples_per_step, 2))] + [edge[n % len(edge)]]
        blocks = {}
        for pj, pi in samples:
            for b in range(max(pj - 1, 0), min(pj + 2, npx)):
                for a in range(max(pi - 1, 0), min(pi + 2, npx)):
                    blocks[(a, b)] = g.read(1, b * npx + a).copy()
        g.fill_ghost(1, n * dt)
        cfl = g.advance_level(1, dt)
        assert cfl == (dt / dx) * 1.0
        for pj, pi in samples:
            js = range(max(pj - 1, 0), min(pj + 2, npx))
            iis = range(max(pi - 1, 0), min(pi + 2, npx))
            dom = (-1 + iis[0] * m * dx, -1 + (iis[-1] + 1) * m * dx,
                   -1 + js[0] * m * dx, -1 + (js[-1] + 1) * m * dx)
            boxes = [(a, b) for b in js for a in iis]
            sub = np.concatenate([W.make_descs([(a - iis[0]) * m], [(b - js[0]) * m], m, m, dx, dx, dom)
                                  for a, b in boxes])
            o = oracle.Oracle(dom, W.EXTRAP, 4, 2, nthreads=1)
            o.set_level(1, sub, np.concatenate([blocks[ab].ravel() for ab in boxes]))
            o.fill_ghost(1, 0.0)
            o.advance_level(1, dt)
            ref = o.read(1, boxes.index((pi, pj)))
            assert rel_err(g.read(1, pj * npx + pi), ref) <= TOL, (n, pi, pj)
            checked += 1
    g.close()
    return checked


def test_c5_full_size_sampled_every_step():
    """C5 (the default bench line's workload and launch configuration), 6
    consecutive steps, 6 sampled blocks per step (edges and corners rotate)."""
    assert sampled_steps(W.c5(), 64, 6, 77, 5) == 36


def test_c4_full_size_sampled_every_step():
    assert sampled_steps(W.c4(), 32, 5, 78, 6) == 35


@pytest.mark.parametrize("name,steps", [("c2", 30), ("c3", 12)])
def test_batched_coarse_steps_equal_single_calls(name, steps):
    """claw_advance_hierarchy_n (K coarse steps per host synchronisation) is
    bitwise the same run as K claw_advance_hierarchy calls, CFLs included,
    and matches the oracle's Berger-Oliger cycles."""
    wl = getattr(W, name)()
    q0s = W.hierarchy_ic(wl)
    nlev = len(wl.levels)
    ratios = [wl.levels[L].ratio for L in range(1, nlev)]
    a = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0)
    b = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0)
    o = oracle.Oracle(wl.domain, wl.bc, wl.limiter, wl.order_trans, nthreads=0)
    for L, (lv, q0) in enumerate(zip(wl.levels, q0s), start=1):
        a.set_level(L, lv.descs, q0)
        b.set_level(L, lv.descs, q0)
        o.set_level(L, lv.descs, q0)
    dt = wl.dt0()
    ca = list(a.advance_hierarchy_n(0.0, dt, 5, update=True)) + \
        list(a.advance_hierarchy_n(5 * dt, dt, steps - 5, update=True))
    ts = [n * dt for n in range(5)] + [5 * dt + k * dt for k in range(steps - 5)]  # the batches' times
    cb = [b.advance_hierarchy(t, dt, update=True) for t in ts]
    co = [oracle_cycle(o, 1, t, dt, nlev, ratios, True) for t in ts]
    assert ca == cb == co
    for L in range(1, nlev + 1):
        assert np.array_equal(a.read_level(L), b.read_level(L))
        assert rel_err(a.read_level(L), o.read_level(L)) <= TOL
    a.close()
    b.close()
