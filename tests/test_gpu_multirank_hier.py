"""Multi-rank hierarchies (claw_config.dist_level): the coarse levels are
replicated on every rank, the finest level is Morton-partitioned.  N virtual
ranks on one GPU (external exchange: same-level halos through claw_halo_pack
/ claw_halo_unpack, the averaged coarse cells through claw_update_pack /
claw_update_unpack), driven level by level in Berger-Oliger order with
updating, must be BITWISE the one-rank claw_advance_hierarchy
run: every rank's replica of each coarse level, each rank's own patches of
the finest, and the coarse-step CFL (max over ranks)."""
import numpy as np
import pytest

from paper_1808_02638_b200 import binding, workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def run_virtual(wl, world, nsteps):
    nlev = len(wl.levels)
    q0s = W.hierarchy_ic(wl)
    ctxs = [binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0, rank=r, world=world, exchange=1,
                         dist_level=nlev) for r in range(world)]
    owners = binding.partition(wl.levels[-1].descs, world)
    offs = W.level_offsets(wl.levels[-1].descs)
    for L, (lv, q) in enumerate(zip(wl.levels, q0s), start=1):
        for r, c in enumerate(ctxs):
            if L < nlev:
                c.set_level(L, lv.descs, q)                       # replicated: every patch
            else:
                mine = [p for p in range(len(lv.descs)) if owners[p] == r]
                c.set_level(L, lv.descs, np.concatenate([q[offs[p]:offs[p + 1]] for p in mine]) if mine
                            else np.zeros(0))
    ratios = [wl.levels[L].ratio for L in range(1, nlev)]

    def cycle(L, t, dt):
        for c in ctxs:
            c.fill_ghost(L, t)
        if L == nlev:
            for r in range(world):
                for s in range(world):
                    if r != s:
                        ctxs[s].halo_unpack(L, r, ctxs[r].halo_pack(L, s))
        cfl = max(c.advance_level(L, dt) for c in ctxs)
        if L < nlev:
            R = ratios[L - 1]
            for k in range(R):
                cfl = max(cfl, cycle(L + 1, t + k * dt / R, dt / R))
            for c in ctxs:
                c.update_level(L + 1)
            if L + 1 == nlev:
                packs = [c.update_pack(L + 1) for c in ctxs]
                for r in range(world):
                    for s in range(world):
                        if r != s:
                            ctxs[s].update_unpack(L + 1, r, packs[r])
        return cfl

    dt = wl.dt0()
    cfls = [cycle(1, n * dt, dt) for n in range(nsteps)]
    return ctxs, owners, offs, cfls


@pytest.mark.parametrize("name,world,nsteps", [("c2", 2, 6), ("c2", 3, 4), ("c3", 2, 3), ("c3", 4, 2)])
def test_replicated_coarse_partitioned_finest_bitwise_equal_single_rank(name, world, nsteps):
    wl = getattr(W, name)()
    nlev = len(wl.levels)
    ctxs, owners, offs, cfls = run_virtual(wl, world, nsteps)
    ref = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0)
    for L, (lv, q) in enumerate(zip(wl.levels, W.hierarchy_ic(wl)), start=1):
        ref.set_level(L, lv.descs, q)
    dt = wl.dt0()
    ref_cfl = [ref.advance_hierarchy(n * dt, dt, update=True) for n in range(nsteps)]
    assert cfls == ref_cfl
    for L in range(1, nlev):
        want = ref.read_level(L)
        for c in ctxs:
            assert np.array_equal(c.read_level(L), want), (L, c.rank)
    full = ref.read_level(nlev)
    nd = len(wl.levels[-1].descs)
    for r, c in enumerate(ctxs):
        want = np.concatenate([full[offs[p]:offs[p + 1]] for p in range(nd) if owners[p] == r])
        assert np.array_equal(c.read_level(nlev), want), r
        assert c.debug_update_counts(nlev, r)[0] > 0
    ref.close()
    for c in ctxs:
        c.close()


def test_dist_level_rules():
    wl = W.c2()
    with pytest.raises(binding.ClawError):
        binding.Claw(wl.domain, wl.bc, 4, 2, device=0, rank=0, world=2, exchange=1, dist_level=1)
    c = binding.Claw(wl.domain, wl.bc, 4, 2, device=0, rank=0, world=2, exchange=1)   # dist_level 0
    c.set_level(1, wl.levels[0].descs)
    with pytest.raises(binding.ClawError):          # level 2 needs dist_level >= 2
        c.set_level(2, wl.levels[1].descs)
    c.close()
