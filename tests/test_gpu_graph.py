"""claw_advance_hierarchy can replay the coarse step as a CUDA graph (SURVEY
8(a) a10; opt-in, CLAW_GRAPH=1).  A replay must be bitwise equal to launching every kernel (the
default path): same data on every level, same CFL, same launch and
cell counts, with updating, with the conservation fix and with profiling on;
re-defining a level or regridding invalidates the captured graphs."""
import os

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


def run(wl, q0s, steps, graphs, reflux=False, profiling=False, update=True):
    old = os.environ.get("CLAW_GRAPH")
    os.environ["CLAW_GRAPH"] = "1" if graphs else "0"
    try:
        g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0, reflux=reflux)
    finally:
        if old is None:
            del os.environ["CLAW_GRAPH"]
        else:
            os.environ["CLAW_GRAPH"] = old
    for L, (lv, q0) in enumerate(zip(wl.levels, q0s), start=1):
        g.set_level(L, lv.descs, q0)
    g.set_profiling(profiling)
    dt = wl.dt0()
    cfl = [g.advance_hierarchy(n * dt, dt, update=update) for n in range(steps)]
    out = [g.read_level(L) for L in range(1, len(wl.levels) + 1)]
    st = g.stats()
    g.close()
    return out, cfl, st


@pytest.mark.parametrize("name,steps,reflux,profiling", [("c2", 7, False, False), ("c3", 5, False, True),
                                                           ("c2", 5, True, False)])
def test_graph_replay_is_bitwise_the_launch_sequence(name, steps, reflux, profiling):
    wl = getattr(W, name)()
    q0s = [W.random_ic(L.descs, 90 + k) for k, L in enumerate(wl.levels)]
    a, ca, sa = run(wl, q0s, steps, True, reflux, profiling)
    b, cb, sb = run(wl, q0s, steps, False, reflux, profiling)
    assert ca == cb
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    for k in ("step_launches", "ghost_launches", "cells_advanced"):
        assert sa[k] == sb[k], k
    if profiling:
        assert sa["step_ms"] > 0 and abs(sa["step_ms"] - sb["step_ms"]) < 0.5 * sb["step_ms"]


def test_graphs_follow_level_changes():
    """Re-setting a level (new buffers) and a regrid drop the captured graphs:
    the run afterwards equals the launch path."""
    wl = W.c2()
    q0s = [W.random_ic(L.descs, 7 + k) for k, L in enumerate(wl.levels)]
    res = []
    for graphs in (True, False):
        os.environ["CLAW_GRAPH"] = "1" if graphs else "0"
        g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0)
        del os.environ["CLAW_GRAPH"]
        for L, (lv, q0) in enumerate(zip(wl.levels, q0s), start=1):
            g.set_level(L, lv.descs, q0)
        dt = wl.dt0()
        for n in range(3):
            g.advance_hierarchy(n * dt, dt)
        g.set_level(2, wl.levels[1].descs, q0s[1])          # new level-2 buffers
        for n in range(3, 5):
            g.advance_hierarchy(n * dt, dt)
        g.regrid(1, [(70, 70, 20, 12), (40, 90, 8, 16)], 4)
        for n in range(5, 8):
            g.advance_hierarchy(n * dt, dt)
        res.append([g.read_level(1), g.read_level(2)])
        g.close()
    for x, y in zip(*res):
        assert np.array_equal(x, y)
