"""GPU regridding (NEXT-3; R18) against the
oracle, through the C-ABI.

Flags are integer decisions taken from fp64 data, so both sides flag the SAME
bytes (the GPU level is overwritten with the oracle's state first): the flag
maps, the clusters and the new levels' patch lists must then be bit-exact,
and the new level's data bitwise equal (copies, and the R10 interpolation in
the same operation order).  Runs continued after a regrid stay within the
north_star bar (1e-12 relative)."""
import numpy as np
import pytest

import oracle
from paper_1808_02638_b200 import binding, workloads as W

pytestmark = pytest.mark.gpu

DOM = (0.0, 1.0, 0.0, 1.0)
TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    binding.load()


def boxes_descs(boxes, R, n1, dom=DOM):
    dxf = (dom[1] - dom[0]) / n1 / R
    return np.concatenate([W.make_descs([a * R], [b * R], w * R, h * R, dxf, dxf, dom) for a, b, w, h in boxes])


def pair(n1, npx, q1, bc=W.EXTRAP, fine=None, dom=DOM, limiter=4, order_trans=2):
    """GPU context and oracle with the same level 1 (n1 x n1 split npx x npx)
    and optional finer levels fine = [(boxes, R, q or None), ...]."""
    d1 = W.uniform_level(npx, npx, n1 // npx, n1 // npx, dom)
    g = binding.Claw(dom, bc, limiter, order_trans, device=0)
    o = oracle.Oracle(dom, bc, limiter, order_trans)
    for h in (g, o):
        h.set_level(1, d1, q1)
    nprev, lev = n1, 1
    for boxes, R, qf in fine or []:
        fd = boxes_descs(boxes, R, nprev, dom)
        q = qf if qf is not None else W.random_ic(fd, 7 + lev)
        for h in (g, o):
            h.set_level(lev + 1, fd, q)
        nprev, lev = nprev * R, lev + 1
    return g, o


def sync(g, o, nlev):
    """Make the GPU's current buffers the oracle's bytes (flags are decisions)."""
    for l in range(1, nlev + 1):
        g.write_level(l, o.read_level(l))


def cover_map(descs, nx, ny, dom=DOM):
    return oracle.cover_map(descs, dom, nx, ny)


nest_mask = oracle.nest_mask


def same_level(g, o, level):
    dg, do = g.descs(level), o.descs(level)
    assert len(dg) == len(do)
    for k in ("mx", "my", "xlower", "ylower", "dx", "dy"):
        assert np.array_equal(dg[k], do[k]), k
    for p in range(len(dg)):
        assert np.array_equal(g.read(level, p), o.read(level, p)), p


@pytest.mark.parametrize("bc", [W.EXTRAP, W.PERIODIC])
@pytest.mark.parametrize("npx", [1, 4])
def test_flag_single_level_equals_oracle(bc, npx):
    rng = np.random.default_rng(3 + npx)
    n = 32
    q = np.round(rng.uniform(-1, 1, (3, n, n)), 1)      # exact ties with tol
    d1 = W.uniform_level(npx, npx, n // npx, n // npx, DOM)
    flat = np.concatenate([q[:, (p // npx) * (n // npx):(p // npx + 1) * (n // npx),
                             (p % npx) * (n // npx):(p % npx + 1) * (n // npx)].ravel() for p in range(len(d1))])
    g = binding.Claw(DOM, bc, 4, 2, device=0)
    o = oracle.Oracle(DOM, bc, 4, 2)
    for h in (g, o):
        h.set_level(1, d1, flat)
        h.fill_ghost(1, 0.0)
    for tol in (0.6, 0.3, 0.0, np.inf):
        fo = o.flag(1, tol)
        assert np.array_equal(g.flag(1, tol), fo)
        for b in (1, 2, 3):
            assert np.array_equal(g.flag(1, tol, buffer=b), oracle.buffer_flags(fo, b))
    g.close()


def test_flag_fine_level_with_coarse_ghosts():
    """Level-2 flags read coarse-interpolated ghosts at a time between the
    coarse level's two time levels; buffered flags clipped to the level
    (clip 1) and to the nesting mask (clip 2)."""
    rng = np.random.default_rng(5)
    n1, R = 24, 2
    g, o = pair(n1, 2, rng.uniform(-1, 1, (3, n1, n1)).ravel(),
                fine=[([(3, 4, 8, 6), (11, 4, 5, 9), (6, 14, 9, 6)], R, None)])
    dt = 0.4 / n1
    for h in (g, o):
        h.fill_ghost(1, 0.0)
        h.advance_level(1, dt)
    sync(g, o, 2)
    t = 0.5 * dt
    for h in (g, o):
        h.fill_ghost(2, t)
    on = cover_map(o.descs(2), n1 * R, n1 * R)
    M = nest_mask(on)
    assert 0 < M.sum() < on.sum()
    for tol in (0.5, 0.9):
        fo = o.flag(2, tol)
        assert fo.sum() > 0
        assert np.array_equal(g.flag(2, tol), fo)
        assert np.array_equal(g.flag(2, tol, buffer=2, clip=1), oracle.buffer_flags(fo, 2, on))
        assert np.array_equal(g.flag(2, tol, buffer=1, clip=2), oracle.buffer_flags(fo, 1, M))
    g.close()


@pytest.mark.parametrize("R", [2, 4])
def test_regrid_without_old_fine_level(R):
    rng = np.random.default_rng(R)
    n1 = 16
    g, o = pair(n1, 2, rng.uniform(-1, 1, (3, n1, n1)).ravel())
    boxes = [(3, 3, 6, 6), (1, 10, 3, 4), (10, 0, 6, 3)]
    for h in (g, o):
        h.regrid(1, boxes, R)
    same_level(g, o, 2)
    g.close()


def test_regrid_copies_old_fine_cells_and_interpolates_the_rest():
    rng = np.random.default_rng(8)
    n1, R = 16, 2
    g, o = pair(n1, 2, rng.uniform(-1, 1, (3, n1, n1)).ravel(), fine=[([(2, 2, 5, 4), (9, 8, 4, 5)], R, None)])
    dt = 0.4 / n1
    for h in (g, o):                                  # one coarse step + its fine steps
        h.fill_ghost(1, 0.0)
        h.advance_level(1, dt)
        for k in range(R):
            h.fill_ghost(2, k * dt / R)
            h.advance_level(2, dt / R)
    sync(g, o, 2)
    new = [(3, 3, 6, 6), (1, 10, 3, 4), (9, 9, 2, 2)]
    for h in (g, o):
        h.regrid(1, new, R)
    same_level(g, o, 2)
    # same boxes again: the data is kept bitwise; no boxes: the level goes
    before = [g.read(2, p) for p in range(3)]
    g.regrid(1, new, R)
    assert all(np.array_equal(g.read(2, p), before[p]) for p in range(3))
    g.regrid(1, [], R)
    assert len(g.descs(2)) == 0
    g.close()


def test_regrid_third_level_from_second():
    rng = np.random.default_rng(11)
    n1 = 16
    g, o = pair(n1, 2, rng.uniform(-1, 1, (3, n1, n1)).ravel(),
                fine=[([(2, 2, 10, 10)], 2, None), ([(6, 6, 8, 6)], 2, None)])
    new = [(6, 6, 4, 4), (10, 12, 6, 5)]
    for h in (g, o):
        h.regrid(2, new, 2)
    same_level(g, o, 3)
    assert len(g.descs(2)) == 1
    # a box whose interpolation needs level-2 cells that do not exist
    for h in (g, o):
        with pytest.raises((binding.ClawError, oracle.OracleError)):
            h.regrid(2, [(0, 0, 4, 4)], 2)
    with pytest.raises(binding.ClawError) as e:
        g.regrid(2, [(30, 30, 4, 4)], 2)               # outside the index space
    assert e.value.code == binding.CLAW_EINVAL
    g.close()


def test_regrid_auto_equals_oracle_composition_and_continues():
    """Ring workload: flag + buffer + cluster + nesting split + regrid in one
    native call (level 1 -> 2, then 2 -> 3) equals the oracle's composition
    step by step; the 3-level run then continues within the parity bar."""
    n1 = 64
    d1 = W.uniform_level(2, 2, 32, 32, W.DOMAIN)
    q1 = W.ring_ic(d1)
    g = binding.Claw(W.DOMAIN, W.EXTRAP, 4, 2, device=0)
    o = oracle.Oracle(W.DOMAIN, W.EXTRAP, 4, 2)
    dt = 0.9 * 2.0 / n1
    for h in (g, o):
        h.set_level(1, d1, q1)
        for k in range(4):
            h.fill_ghost(1, k * dt)
            h.advance_level(1, dt)
    sync(g, o, 1)
    t = o.level_time(1)[1]
    cfg = dict(tol=0.05, buffer=2, cutoff=0.7, max_dim=16, min_dim=4)

    def oracle_auto(level, R):
        o.fill_ghost(level, t)
        return oracle.regrid_auto(o, level, R=R, **cfg)

    g.fill_ghost(1, t)
    nb = g.regrid_auto(1, R=4, **cfg)
    assert nb == oracle_auto(1, 4) and nb > 4
    same_level(g, o, 2)
    g.fill_ghost(2, t)
    nb = g.regrid_auto(2, R=2, **cfg)
    assert nb == oracle_auto(2, 2) and nb > 4
    same_level(g, o, 3)
    ratios = {1: 4, 2: 2}
    for k in range(3):                                 # Berger-Oliger cycles
        binding.berger_oliger(g, 1, t + k * dt, dt, ratios, 3)
        _bo_oracle(o, 1, t + k * dt, dt, ratios, 3)
    for l in (1, 2, 3):
        qg, qo = g.read_level(l), o.read_level(l)
        assert np.abs(qg - qo).max() <= TOL * np.abs(qo).max(), l
    g.close()


def _bo_oracle(o, level, t, dt, ratios, nlev):
    o.fill_ghost(level, t)
    o.advance_level(level, dt)
    if level < nlev:
        R = ratios[level]
        for k in range(R):
            _bo_oracle(o, level + 1, t + k * dt / R, dt / R, ratios, nlev)


def test_regrid_reuses_pool_blocks():
    rng = np.random.default_rng(2)
    n1 = 32
    g, _ = pair(n1, 2, rng.uniform(-1, 1, (3, n1, n1)).ravel())
    for k in range(2):                                  # the second regrid frees the first level's blocks
        g.regrid(1, [(4, 4, 12, 12)], 4)
    s0 = binding.pool_stats()
    for k in range(4):
        g.regrid(1, [(4 + k, 4, 12, 12)], 4)            # same sizes: every block comes from the pool
    s1 = binding.pool_stats()
    assert s1["misses"] == s0["misses"] and s1["hits"] > s0["hits"]
    g.close()


def test_regrid_in_turn_keeps_every_levels_data():
    """R18: regrid(1) then regrid(2) copy both finer levels' old data (the
    level 3 discarded by the first regrid is the second one's copy source),
    as the oracle does; new boxes mix copied and interpolated cells."""
    rng = np.random.default_rng(21)
    n1 = 16
    g, o = pair(n1, 2, rng.uniform(-1, 1, (3, n1, n1)).ravel(),
                fine=[([(3, 3, 10, 9)], 2, None), ([(8, 8, 10, 8)], 2, None)])
    q3 = g.read(3, 0)
    for h in (g, o):
        h.regrid(1, [(3, 3, 10, 9)], 2)
        h.regrid(2, [(8, 8, 10, 8)], 2)
    assert np.array_equal(g.read(3, 0), q3)
    for h in (g, o):
        h.regrid(1, [(2, 3, 11, 10)], 2)
        h.regrid(2, [(7, 9, 12, 6), (9, 16, 5, 3)], 2)
    same_level(g, o, 2)
    same_level(g, o, 3)
    g.close()
