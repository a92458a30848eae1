"""Pins of the oracle's regridding (NEXT-3; R18):
flagging, flag buffering, Berger-Rigoutsos clustering and the new level's
initial data.  Fixed by the SPEC's worked examples, brute-force evaluation
of the flag criterion in numpy, scipy's maximum filter for the dilation,
the clustering postconditions, and closed forms of the interpolation."""
import numpy as np
import pytest
from scipy import ndimage

import oracle
from paper_1808_02638_b200 import workloads as W


def one_level(q, dom=(0.0, 1.0, 0.0, 1.0), bc=W.EXTRAP, npx=1, npy=1):
    """A single level holding the [3, ny, nx] field q, split npx x npy."""
    _, ny, nx = q.shape
    d = W.uniform_level(npx, npy, nx // npx, ny // npy, dom)
    flat = []
    for p in range(len(d)):
        i0, j0 = (p % npx) * (nx // npx), (p // npx) * (ny // npy)
        flat.append(q[:, j0:j0 + ny // npy, i0:i0 + nx // npx].ravel())
    o = oracle.Oracle(dom, bc, 4, 2)
    o.set_level(1, d, np.concatenate(flat))
    o.fill_ghost(1, 0.0)
    return o


def brute_flags(p, tol, periodic=False):
    """max over the 4 edge neighbours of |p_n - p| > tol, neighbours by the
    composite rule (clamp = extrapolation, or wrap)."""
    mode = "wrap" if periodic else "edge"
    pp = np.pad(p, 1, mode=mode)
    c = pp[1:-1, 1:-1]
    g = np.maximum.reduce([np.abs(pp[1:-1, :-2] - c), np.abs(pp[1:-1, 2:] - c),
                           np.abs(pp[:-2, 1:-1] - c), np.abs(pp[2:, 1:-1] - c)])
    return (g > tol).astype(np.uint8)


def test_flag_examples():
    q = np.zeros((3, 12, 12))
    q[0, 5, 5] = 1.0                                # spike of height 1 at (5,5), tol 0.5
    f = one_level(q).flag(1, 0.5)
    want = np.zeros((12, 12), np.uint8)
    for i, j in [(5, 5), (4, 5), (6, 5), (5, 4), (5, 6)]:
        want[j, i] = 1
    assert np.array_equal(f, want)
    assert not one_level(np.full((3, 12, 12), 0.3)).flag(1, 0.0).any()     # constant field
    assert not one_level(q).flag(1, np.inf).any()                           # tol = inf


@pytest.mark.parametrize("periodic", [False, True])
def test_flag_brute_force_and_tiling(periodic):
    rng = np.random.default_rng(4)
    q = rng.uniform(-1, 1, (3, 24, 32))
    q[0] = np.round(q[0], 1)                          # exact ties with tol
    bc = W.PERIODIC if periodic else W.EXTRAP
    want = brute_flags(q[0], 0.6, periodic)
    assert 0 < want.sum() < want.size
    for npx, npy in [(1, 1), (4, 3), (2, 2)]:
        assert np.array_equal(one_level(q, bc=bc, npx=npx, npy=npy).flag(1, 0.6), want)


def test_buffer_examples_and_scipy():
    e = np.zeros((11, 11), np.uint8)
    assert not oracle.buffer_flags(e, 2).any()
    e[5, 5] = 1
    b1 = oracle.buffer_flags(e, 1)
    assert b1.sum() == 9 and b1[4:7, 4:7].all()      # 3x3 block
    assert np.array_equal(oracle.buffer_flags(e, 0), e)
    rng = np.random.default_rng(1)
    f = (rng.uniform(size=(37, 53)) > 0.97).astype(np.uint8)
    for b in (1, 2, 3):
        want = ndimage.maximum_filter(f, size=2 * b + 1, mode="constant", cval=0)
        assert np.array_equal(oracle.buffer_flags(f, b), want)
    mask = (rng.uniform(size=f.shape) > 0.3).astype(np.uint8)
    assert np.array_equal(oracle.buffer_flags(f, 2, mask),
                          ndimage.maximum_filter(f, size=5, mode="constant") & mask)


def check_boxes(f, boxes, cutoff, max_dim, min_dim):
    cover = np.zeros(f.shape, np.int32)
    for i0, j0, w, h in boxes:
        assert w >= 1 and h >= 1 and w <= max_dim and h <= max_dim
        blk = f[j0:j0 + h, i0:i0 + w]
        # tight: every edge row / column of the box holds a flag
        assert blk[0].any() and blk[-1].any() and blk[:, 0].any() and blk[:, -1].any()
        eff = blk.sum() / (w * h)
        assert eff >= cutoff or max(w, h) < 2 * min_dim
        cover[j0:j0 + h, i0:i0 + w] += 1
    assert cover.max() <= 1                           # disjoint
    assert (cover[f == 1] == 1).all()                 # every flag covered exactly once


def test_cluster_examples():
    f = np.zeros((20, 30), np.uint8)
    f[2:12, 3:13] = 1                                  # one box, efficiency 1
    assert oracle.cluster(f, 0.9, 64, 2).tolist() == [[3, 2, 10, 10]]
    g = np.zeros((10, 30), np.uint8)
    g[2:6, 2:6] = 1
    g[2:6, 16:20] = 1                                  # two blocks, 10-cell gap
    b = oracle.cluster(g, 0.7, 64, 2)
    assert sorted(map(tuple, b.tolist())) == [(2, 2, 4, 4), (16, 2, 4, 4)]
    assert len(oracle.cluster(np.zeros((8, 8), np.uint8), 0.7, 16, 2)) == 0


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("cutoff,max_dim,min_dim", [(0.7, 32, 4), (0.9, 16, 2), (0.5, 64, 8)])
def test_cluster_postconditions_random(seed, cutoff, max_dim, min_dim):
    rng = np.random.default_rng(seed)
    # a ring-like flag set plus noise
    ny, nx = 70, 90
    Y, X = np.mgrid[0:ny, 0:nx]
    r = np.hypot(X - 40 - seed, Y - 33)
    f = ((np.abs(r - 22) < 3) | (rng.uniform(size=(ny, nx)) > 0.995)).astype(np.uint8)
    b = oracle.cluster(f, cutoff, max_dim, min_dim)
    check_boxes(f, b, cutoff, max_dim, min_dim)
    assert np.array_equal(b, oracle.cluster(f, cutoff, max_dim, min_dim))     # deterministic


def two_levels(q1, fine_boxes, R, dom=(0.0, 1.0, 0.0, 1.0), bc=W.EXTRAP, qf=None):
    _, ny, nx = q1.shape
    o = oracle.Oracle(dom, bc, 4, 2)
    o.set_level(1, W.uniform_level(1, 1, nx, ny, dom), q1.ravel())
    if fine_boxes:
        dxf = (dom[1] - dom[0]) / nx / R
        fd = np.concatenate([W.make_descs([a * R], [b * R], w * R, h * R, dxf, dxf, dom)
                             for a, b, w, h in fine_boxes])
        o.set_level(2, fd, qf if qf is not None else W.random_ic(fd, 3))
    return o


def test_regrid_copy_and_interpolation():
    rng = np.random.default_rng(8)
    n, R = 16, 4
    q1 = rng.uniform(-1, 1, (3, n, n))
    old = [(2, 2, 5, 4), (9, 8, 4, 5)]
    o = two_levels(q1, old, R)
    old_fine = {p: o.read(2, p) for p in range(2)}
    new = [(3, 3, 6, 6), (1, 10, 3, 4)]
    o.regrid(1, new, R)
    d = o.descs(2)
    assert len(d) == 2 and list(d["mx"]) == [24, 12] and list(d["my"]) == [24, 16]
    for p, (a, b, w, h) in enumerate(new):
        q = o.read(2, p)
        for jj in range(h * R):
            for ii in range(w * R):
                I, J = a * R + ii, b * R + jj
                src = None
                for op, (oa, ob, ow, oh) in enumerate(old):
                    if oa * R <= I < (oa + ow) * R and ob * R <= J < (ob + oh) * R:
                        src = old_fine[op][:, J - ob * R, I - oa * R]
                if src is not None:
                    assert np.array_equal(q[:, jj, ii], src)             # copied from the old level 2
        # interpolated coarse cells (no old fine cell inside): mean of children = coarse value
        for cj in range(h):
            for ci in range(w):
                Ic, Jc = a + ci, b + cj
                blk = q[:, cj * R:(cj + 1) * R, ci * R:(ci + 1) * R]
                overlap = any(oa <= Ic < oa + ow and ob <= Jc < ob + oh for oa, ob, ow, oh in old)
                if not overlap:
                    assert np.allclose(blk.mean(axis=(1, 2)), q1[:, Jc, Ic], rtol=0, atol=1e-15)


def test_regrid_linear_field_exact_and_same_boxes_identity():
    n, R = 16, 2
    Y, X = np.mgrid[0:n, 0:n]
    q1 = np.stack([0.5 + 0.25 * X - 0.125 * Y, 1.0 + 0.0625 * X, -0.5 * Y])   # dyadic linear field
    o = two_levels(q1, [], R)
    o.regrid(1, [(4, 4, 6, 5)], R)
    q = o.read(2, 0)
    fx = (np.arange(12) + 0.5) / R + 4 - 0.5       # fine centres in coarse index units
    fy = (np.arange(10) + 0.5) / R + 4 - 0.5
    FX, FY = np.meshgrid(fx, fy)
    want = np.stack([0.5 + 0.25 * FX - 0.125 * FY, 1.0 + 0.0625 * FX, -0.5 * FY])
    assert np.array_equal(q, want)
    # regridding onto the same boxes keeps the fine data bitwise
    o2 = two_levels(np.random.default_rng(2).uniform(-1, 1, (3, n, n)), [(3, 3, 4, 4)], R)
    before = o2.read(2, 0)
    o2.regrid(1, [(3, 3, 4, 4)], R)
    assert np.array_equal(o2.read(2, 0), before)
    # no boxes: the fine level is removed
    o2.regrid(1, [], R)
    assert len(o2.descs(2)) == 0


def test_regrid_not_nested_fails():
    n, R = 16, 2
    o = two_levels(np.zeros((3, n, n)), [(2, 2, 8, 8)], R)
    o.regrid(1, [(2, 2, 8, 8)], R)
    # level 3 from level 2: a box outside level 2 has no coarse donor
    with pytest.raises(oracle.OracleError):
        o.regrid(2, [(0, 0, 4, 4)], 2)


def test_ring_regrid_covers_every_flag():
    """after flag + buffer + cluster + regrid, every buffered flagged
    coarse cell lies inside the new fine level."""
    wl = W.c2()
    d1 = wl.levels[0].descs
    o = oracle.Oracle(wl.domain, wl.bc, 4, 2)
    o.set_level(1, d1, W.ring_ic(d1))
    dt = wl.dt0()
    for k in range(5):                                 # let the ring move
        o.fill_ghost(1, k * dt)
        o.advance_level(1, dt)
    o.fill_ghost(1, 5 * dt)
    f = oracle.buffer_flags(o.flag(1, 0.05), 2)
    assert f.sum() > 100
    boxes = oracle.cluster(f, 0.7, 32, 4)
    check_boxes(f, boxes, 0.7, 32, 4)
    o.regrid(1, boxes, 4)
    d2 = o.descs(2)
    cov = np.zeros(f.shape, bool)
    for e in d2:
        i0 = int(round((e["xlower"] - wl.domain[0]) / e["dx"])) // 4
        j0 = int(round((e["ylower"] - wl.domain[2]) / e["dy"])) // 4
        cov[j0:j0 + e["my"] // 4, i0:i0 + e["mx"] // 4] = True
    assert cov[f == 1].all()


def brute_nest_mask(on):
    ny, nx = on.shape
    M = np.zeros_like(on)
    for J in range(ny):
        for I in range(nx):
            blk = on[max(J - 2, 0):J + 3, max(I - 2, 0):I + 3]
            M[J, I] = 1 if on[J, I] and blk.all() else 0
    return M


@pytest.mark.parametrize("seed", range(4))
def test_nest_mask_brute_force(seed):
    rng = np.random.default_rng(40 + seed)
    on = np.zeros((30, 37), np.uint8)
    for _ in range(6):
        a, b = rng.integers(0, 30), rng.integers(0, 25)
        on[b:b + rng.integers(3, 15), a:a + rng.integers(3, 15)] = 1
    assert np.array_equal(oracle.nest_mask(on), brute_nest_mask(on))
    full = np.ones((9, 11), np.uint8)
    assert oracle.nest_mask(full).all()                 # the domain edge never vetoes


@pytest.mark.parametrize("seed", range(6))
def test_split_boxes_postconditions(seed):
    rng = np.random.default_rng(60 + seed)
    on = np.zeros((50, 60), np.uint8)
    for _ in range(5):
        a, b = rng.integers(0, 50), rng.integers(0, 40)
        on[b:b + rng.integers(5, 25), a:a + rng.integers(5, 25)] = 1
    M = oracle.nest_mask(on)
    f = ((rng.uniform(size=on.shape) > 0.8) & (M == 1)).astype(np.uint8)
    f = oracle.buffer_flags(f, 1, M)
    boxes = oracle.cluster(f, 0.6, 24, 3)
    pieces = oracle.split_boxes(boxes, M, f)
    cover = np.zeros(on.shape, np.int32)
    for x0, y0, w, h in pieces:
        blk = M[y0:y0 + h, x0:x0 + w]
        assert blk.all()                                 # inside the nesting mask
        assert f[y0:y0 + h, x0:x0 + w].any()             # holds a flag
        assert any(bx <= x0 and x0 + w <= bx + bw and by <= y0 and y0 + h <= by + bh
                   for bx, by, bw, bh in boxes)           # inside one cluster box
        cover[y0:y0 + h, x0:x0 + w] += 1
    assert cover.max() <= 1 and (cover[f == 1] == 1).all()


def test_regrid_in_turn_keeps_every_levels_data():
    """R18: regridding level 1, then level 2, onto the same boxes keeps levels
    2 and 3 bitwise (the level-3 data discarded by the first regrid is the copy
    source of the second); once a level advances, the discarded data is gone
    and level 3 is interpolated from level 2."""
    n, R = 16, 2
    rng = np.random.default_rng(12)
    dom = (0.0, 1.0, 0.0, 1.0)
    o = oracle.Oracle(dom, W.EXTRAP, 4, 2)
    o.set_level(1, W.uniform_level(1, 1, n, n, dom), rng.uniform(-1, 1, 3 * n * n))
    b2, b3 = [(3, 3, 10, 9)], [(8, 8, 10, 8)]
    d2 = np.concatenate([W.make_descs([a * R], [b * R], w * R, h * R, 1 / n / R, 1 / n / R, dom) for a, b, w, h in b2])
    d3 = np.concatenate([W.make_descs([a * R], [b * R], w * R, h * R, 1 / n / R / R, 1 / n / R / R, dom)
                         for a, b, w, h in b3])
    o.set_level(2, d2, W.random_ic(d2, 1))
    o.set_level(3, d3, W.random_ic(d3, 2))
    q2, q3 = o.read(2, 0), o.read(3, 0)
    o.regrid(1, b2, R)
    assert len(o.descs(3)) == 0
    o.regrid(2, b3, R)
    assert np.array_equal(o.read(2, 0), q2) and np.array_equal(o.read(3, 0), q3)
    o.regrid(1, b2, R)
    o.fill_ghost(1, 0.0)
    o.advance_level(1, 0.0)                 # time moves (dt = 0): the discarded level 3 is dropped
    o.regrid(2, b3, R)
    assert not np.array_equal(o.read(3, 0), q3)
