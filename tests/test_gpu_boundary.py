"""The C-ABI boundary's device-memory and debug contract:

* claw_config.arena: a context created on device memory PyTorch owns carves
  every buffer from it (the paper's pool, with the ownership on the
  caller's side) -- results bitwise those of the library's own pool, no
  cudaMalloc for the context, CLAW_ENOMEM (not sticky) when the arena is full;
* claw_config.check_finite: CLAW_ENONFINITE after a step that
  produced NaN / Inf, nothing otherwise.
"""
import numpy as np
import pytest

import oracle
from paper_1808_02638_b200 import binding, workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    t = pytest.importorskip("torch")
    if not t.cuda.is_available():
        pytest.skip("no CUDA device")
    binding.load()
    return t


def run(g, wl, q0, nsteps):
    descs = wl.levels[0].descs
    g.set_level(1, descs, q0)
    dt = wl.dt0()
    cfl = []
    for n in range(nsteps):
        g.fill_ghost(1, n * dt)
        cfl.append(g.advance_level(1, dt))
    return g.read_level(1), cfl


@pytest.mark.parametrize("name", ["c1", "c5_reduced", "c3"])
def test_level_inside_a_torch_arena_is_bitwise_the_pool_run(torch, name):
    if name == "c3":
        wl = W.c3()
    else:
        wl = W.c1() if name == "c1" else W.c5(16, 64)   # 1024^2 cells of 64^2 patches
    arena = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    pool0 = binding.pool_stats()
    a = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0, arena=arena)
    if name == "c3":
        dt = wl.dt0()
        for L, (lv, q) in enumerate(zip(wl.levels, W.hierarchy_ic(wl)), start=1):
            a.set_level(L, lv.descs, q)
        ca = [a.advance_hierarchy(n * dt, dt, update=True) for n in range(3)]
    else:
        q0 = W.ring_ic(wl.levels[0].descs)
        qa, ca = run(a, wl, q0, 20)
    pool1 = binding.pool_stats()
    # nothing of the arena context came from the library's own pool
    assert (pool1["hits"], pool1["misses"]) == (pool0["hits"], pool0["misses"])
    b = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0)
    if name == "c3":
        for L, (lv, q) in enumerate(zip(wl.levels, W.hierarchy_ic(wl)), start=1):
            b.set_level(L, lv.descs, q)
        assert ca == [b.advance_hierarchy(n * dt, dt, update=True) for n in range(3)]
        for L in range(1, 4):
            assert np.array_equal(a.read_level(L), b.read_level(L))
    else:
        qb, cb = run(b, wl, q0, 20)
        assert ca == cb
        assert np.array_equal(qa, qb)
        if name == "c1":
            o = oracle.Oracle(wl.domain, wl.bc, wl.limiter, wl.order_trans)
            o.set_level(1, wl.levels[0].descs, q0)
            for n in range(20):
                o.fill_ghost(1, n * wl.dt0())
                o.advance_level(1, wl.dt0())
            ref = o.read_level(1)
            assert np.abs(qa - ref).max() <= 1e-12 * np.abs(ref).max()
    # the arena context's device buffers lie inside the arena
    _, cells, dev_bytes = a.level_owned(1)
    assert 0 < dev_bytes <= arena.numel()
    a.close()
    b.close()
    del arena


def test_arena_full_is_enomem_and_not_sticky(torch):
    arena = torch.empty(4 << 20, dtype=torch.uint8, device="cuda")   # 4 MiB
    g = binding.Claw(W.DOMAIN, W.EXTRAP, 4, 2, device=0, arena=arena)
    big = W.uniform_level(8, 8, 64, 64)      # 2 x 6.3 MB of state: does not fit
    with pytest.raises(binding.ClawError) as e:
        g.set_level(1, big, None)
    assert e.value.code == binding.CLAW_ENOMEM
    wl = W.c1()                               # 2 x 98 KB: fits; the context still works
    q, cfl = run(g, wl, W.ring_ic(wl.levels[0].descs), 3)
    assert cfl[-1] == pytest.approx(0.9)
    g.close()


def test_arena_must_be_device_memory(torch):
    host = torch.empty(1 << 20, dtype=torch.uint8)
    with pytest.raises(binding.ClawError) as e:
        binding.Claw(W.DOMAIN, W.EXTRAP, 4, 2, device=0, arena=(host.data_ptr(), host.numel()))
    assert e.value.code == binding.CLAW_EINVAL


def test_check_finite_flags_a_nan_step(torch):
    wl = W.c1()
    d = wl.levels[0].descs
    g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0, check_finite=True)
    q0 = W.ring_ic(d)
    q, cfl = run(g, wl, q0, 3)                # finite: no error
    bad = q.copy()
    bad[1234] = np.nan
    g.write_level(1, bad)
    g.fill_ghost(1, 0.0)
    with pytest.raises(binding.ClawError) as e:
        g.advance_level(1, wl.dt0())
    assert e.value.code == binding.CLAW_ENONFINITE and "level 1" in str(e.value)
    g.write_level(1, q0)                      # not sticky: a finite state steps again
    g.fill_ghost(1, 0.0)
    assert g.advance_level(1, wl.dt0()) == pytest.approx(0.9)
    g.close()


def test_check_finite_in_the_hierarchy_driver(torch):
    wl = W.c2()
    g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0, check_finite=True)
    qs = W.hierarchy_ic(wl)
    for L, (lv, q) in enumerate(zip(wl.levels, qs), start=1):
        g.set_level(L, lv.descs, q)
    dt = wl.dt0()
    g.advance_hierarchy(0.0, dt, update=True)
    q2 = g.read_level(2)
    q2[17] = np.inf
    g.write_level(2, q2)
    with pytest.raises(binding.ClawError) as e:
        g.advance_hierarchy(dt, dt, update=True)
    assert e.value.code == binding.CLAW_ENONFINITE
    g.close()
