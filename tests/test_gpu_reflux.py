"""Conservation fix (NEXT-2) on the GPU vs the oracle, through the C-ABI.

* the register tables (which coarse cells, which edges, which fine cells) are
  identical to the oracle's -- checked without a GPU on a host-only context;
* register values after the coarse step and after each fine sub-step, and the
  whole hierarchy after several Berger-Oliger cycles with updating + fix,
  agree with the oracle to 1e-12 (the fix re-evaluates edge fluxes, so its
  rounding differs from the oracle's by a few ulps of O(1) terms);
* the GPU's own level-1 totals are conserved to rounding with periodic BCs.
"""
import numpy as np
import pytest

import oracle
from paper_1808_02638_b200 import binding, workloads as W
from test_oracle_reflux import L2_BOXES, L3_BOXES, PER, cycle, hierarchy

TOL = 1e-12
DOM = (-1.0, 1.0, -1.0, 1.0)


def both(levels_boxes, ratios, seed, limiter=4, order_trans=2, bc=PER, device=0):
    descs = hierarchy(levels_boxes, ratios)
    g = binding.Claw(DOM, bc, limiter, order_trans, device=device, reflux=True)
    o = oracle.Oracle(DOM, bc, limiter, order_trans, reflux=True)
    rng = np.random.default_rng(seed)
    for L, d in enumerate(descs, start=1):
        q = rng.uniform(-1, 1, 3 * int((d["mx"] * d["my"]).sum())) if device >= 0 else None
        g.set_level(L, d, q)
        o.set_level(L, d, q)
    return g, o, descs


def test_register_tables_match_oracle_host_only():
    for lb, ra in (([L2_BOXES], [2]), ([L2_BOXES, L3_BOXES], [2, 2])):
        g, o, descs = both(lb, ra, 0, device=-1)
        for L in range(2, len(descs) + 1):
            eg, _ = g.reflux_registers(L, values=False)
            eo, _ = o.reflux_registers(L)
            assert len(eg) > 0 and np.array_equal(eg, eo)


def test_reflux_rejects_unaligned_and_multirank():
    descs = hierarchy([[(17, 20, 8, 8)]], [2])
    g = binding.Claw(DOM, PER, 4, 2, device=-1, reflux=True)
    g.set_level(1, descs[0])
    with pytest.raises(binding.ClawError) as e:
        g.set_level(2, descs[1])
    assert e.value.code == binding.CLAW_EINVAL
    with pytest.raises(binding.ClawError):
        binding.Claw(DOM, PER, 4, 2, device=-1, reflux=True, world=2, rank=0, exchange=1)


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    binding.load()


@pytest.mark.gpu
@pytest.mark.parametrize("limiter,order_trans", [(4, 2), (1, 1), (0, 0), (3, 2), (2, 2)])
def test_register_values_match_oracle(gpu, limiter, order_trans):
    g, o, descs = both([L2_BOXES], [2], 5, limiter, order_trans)
    dt = (0.8 if order_trans else 0.4) * float(descs[0]["dx"][0])
    for h in (g, o):
        h.fill_ghost(1, 0.0)
        h.advance_level(1, dt)
    _, ag = g.reflux_registers(2)
    _, ao = o.reflux_registers(2)
    assert np.abs(ao).max() > 1e-3 and rel(ag, ao) <= TOL
    for k in range(2):
        for h in (g, o):
            h.fill_ghost(2, k * dt / 2)
            h.advance_level(2, dt / 2)
        _, ag = g.reflux_registers(2)
        _, ao = o.reflux_registers(2)
        assert np.abs(ag - ao).max() <= TOL * max(np.abs(ao).max(), 1.0), (k, np.abs(ag - ao).max())
    for h in (g, o):
        h.update_level(2)
    assert rel(g.read_level(1), o.read_level(1)) <= TOL
    _, ag = g.reflux_registers(2)
    assert not ag.any()                 # cleared by the fix


@pytest.mark.gpu
@pytest.mark.parametrize("nlev", [2, 3])
def test_hierarchy_cycles_match_oracle_and_conserve(gpu, nlev):
    lb, ra = [L2_BOXES, L3_BOXES][:nlev - 1], [2, 2][:nlev - 1]
    g, o, descs = both(lb, ra, 9)
    dt = 0.8 * float(descs[0]["dx"][0])
    totals = []
    for n in range(8):
        cycle(o, 1, n * dt, dt, nlev, ra)
        g.advance_hierarchy(n * dt, dt, update=True)      # native driver; update applies the fix
        q1 = g.read_level(1)
        totals.append(q1.reshape(4, 3, -1).sum(axis=(0, 2)))
    for L in range(1, nlev + 1):
        assert rel(g.read_level(L), o.read_level(L)) <= TOL, L
    scale = np.abs(g.read_level(1)).sum()
    drift = np.abs(np.array(totals[1:]) - totals[0]).max()
    assert drift <= 1e-13 * scale, (drift, scale)


@pytest.mark.gpu
def test_c2_with_reflux_matches_oracle(gpu):
    """C2 (extrapolation BCs, R=4, 52 fine patches): 10 coarse steps with
    updating and the conservation fix, GPU vs oracle."""
    wl = W.c2()
    q0s = W.hierarchy_ic(wl)
    g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0, reflux=True)
    o = oracle.Oracle(wl.domain, wl.bc, wl.limiter, wl.order_trans, reflux=True)
    for L, (lv, q0) in enumerate(zip(wl.levels, q0s), start=1):
        g.set_level(L, lv.descs, q0)
        o.set_level(L, lv.descs, q0)
    assert len(g.reflux_registers(2, values=False)[0]) > 0
    dt = wl.dt0()
    for n in range(10):
        g.advance_hierarchy(n * dt, dt, update=True)
        cycle(o, 1, n * dt, dt, 2, [4])
    for L in (1, 2):
        assert rel(g.read_level(L), o.read_level(L)) <= TOL
