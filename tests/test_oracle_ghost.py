"""Pins of the oracle's ghost fill: the three cases of P:125-132 (physical BC,
same-level copy, coarse interpolation), checked against closed forms."""
import numpy as np
import pytest

import oracle
from paper_1808_02638_b200 import workloads as W


def global_field(descs, fn):
    """q[p][m][j][i] = fn(m, I, J) with (I, J) the global cell index."""
    out = []
    for d in descs:
        i0 = int(round((d["xlower"] + 1) / d["dx"]))
        j0 = int(round((d["ylower"] + 1) / d["dy"]))
        J, I = np.meshgrid(np.arange(j0, j0 + d["my"]), np.arange(i0, i0 + d["mx"]), indexing="ij")
        out.append(np.stack([fn(m, I, J) for m in range(3)]).ravel())
    return np.concatenate(out)


@pytest.mark.parametrize("bc", [W.EXTRAP, W.PERIODIC, (1, 1, 2, 2)])
def test_same_level_and_bc_ghosts_closed_form(bc):
    d = W.ragged_level(7, 30, 26, 9)
    nx, ny = 30, 26
    fn = lambda m, I, J: 1e6 * m + 1000.0 * J + I
    o = oracle.Oracle(W.DOMAIN, bc, 4, 2, nthreads=2)
    o.set_level(1, d, global_field(d, fn))
    o.fill_ghost(1, 0.0)
    for p, dd in enumerate(d):
        i0 = int(round((dd["xlower"] + 1) / dd["dx"]))
        j0 = int(round((dd["ylower"] + 1) / dd["dy"]))
        qp = o.read_padded(1, p)
        mx, my = int(dd["mx"]), int(dd["my"])
        for jj in range(my + 4):
            for ii in range(mx + 4):
                I, J = i0 + ii - 2, j0 + jj - 2
                I = (I % nx) if bc[0] == 2 else min(max(I, 0), nx - 1)
                J = (J % ny) if bc[2] == 2 else min(max(J, 0), ny - 1)
                for m in range(3):
                    assert qp[m, jj, ii] == fn(m, I, J)


def test_outflow_edge_value():
    # edge value 7.5 -> both ghost layers 7.5
    q = np.zeros((3, 3, 4))
    q[0, :, -1] = 7.5
    o = oracle.Oracle((0, 4, 0, 3), W.EXTRAP, 4, 2)
    o.set_level(1, W.make_descs([0], [0], 4, 3, 1.0, 1.0, (0, 4, 0, 3)), q.ravel())
    o.fill_ghost(1)
    qp = o.read_padded(1, 0)
    assert (qp[0, 2:5, 6:8] == 7.5).all()


def two_level(R, fine_boxes, coarse_n=8, domain=(0.0, 1.0, 0.0, 1.0), bc=W.EXTRAP):
    dxc = (domain[1] - domain[0]) / coarse_n
    cd = W.uniform_level(1, 1, coarse_n, coarse_n, domain)
    dxf = dxc / R
    fd = np.concatenate([W.make_descs([a], [b], w, h, dxf, dxf, domain)
                         for a, b, w, h in fine_boxes])
    o = oracle.Oracle(domain, bc, 4, 2)
    return o, cd, fd, dxc, dxf


@pytest.mark.parametrize("R", [2, 4])
def test_coarse_interp_reproduces_linear_field_in_time(R):
    """Case 3: a linear field 2x+3y is reproduced exactly at fine cell
    centres, at both bracketing times and in between (linear in time)."""
    o, cd, fd, dxc, dxf = two_level(R, [(2 * R, 2 * R, 2 * R, 2 * R), (5 * R, 5 * R, R, R)])
    n = 8
    xc = (np.arange(n) + 0.5) * dxc
    X, Y = np.meshgrid(xc, xc)
    lin0 = 2 * X + 3 * Y
    lin1 = -1 * X + 0.5 * Y + 0.25
    q0 = np.stack([lin0, lin0 + 1, 2 * lin0]).ravel()
    o.set_level(1, cd, q0)
    o.set_level(2, fd, np.zeros(3 * int((fd["mx"] * fd["my"]).sum())))
    # advance level 1 with dt = 0 and overwrite its new state: t_old=0, t_new=0.5
    o.fill_ghost(1, 0.0)
    o.advance_level(1, 0.5)
    o.write(1, 0, np.stack([lin1, lin1 + 1, 2 * lin1]))
    # level 1 now holds q_old = lin0-fields (t=0) and q_new = lin1-fields (t=0.5)
    for t, a in ((0.0, 0.0), (0.25, 0.5), (0.5, 1.0)):
        o.fill_ghost(2, t)
        for p, d in enumerate(fd):
            qp = o.read_padded(2, p)
            i0 = d["xlower"] / dxf
            j0 = d["ylower"] / dxf
            for jj in range(int(d["my"]) + 4):
                for ii in range(int(d["mx"]) + 4):
                    if 2 <= ii < d["mx"] + 2 and 2 <= jj < d["my"] + 2:
                        continue
                    x = (i0 + ii - 2 + 0.5) * dxf
                    y = (j0 + jj - 2 + 0.5) * dxf
                    f = (1 - a) * (2 * x + 3 * y) + a * (-1 * x + 0.5 * y + 0.25)
                    assert qp[0, jj, ii] == pytest.approx(f, abs=1e-14)
                    assert qp[1, jj, ii] == pytest.approx(f + 1, abs=1e-14)
                    assert qp[2, jj, ii] == pytest.approx(2 * f, abs=1e-14)


@pytest.mark.parametrize("R", [2, 4])
def test_coarse_interp_time_weight(R):
    """alpha = (t - t_old)/(t_new - t_old): with a constant coarse state c0 at
    t_old and c1 at t_new, fine ghosts get (1-alpha) c0 + alpha c1."""
    o, cd, fd, dxc, dxf = two_level(R, [(2 * R, 2 * R, 2 * R, 2 * R)])
    c0 = np.ones(3 * 64) * 2.0
    o.set_level(1, cd, c0)
    o.set_level(2, fd, np.zeros(3 * int((fd["mx"] * fd["my"]).sum())))
    o.fill_ghost(1, 0.0)
    o.advance_level(1, 0.4)            # constant state stays constant; t: 0 -> 0.4
    o.write(1, 0, np.ones((3, 8, 8)) * 6.0)
    for t, expect in ((0.0, 2.0), (0.1, 3.0), (0.2, 4.0), (0.4, 6.0)):
        o.fill_ghost(2, t)
        qp = o.read_padded(2, 0)
        ring = np.ones_like(qp[0], dtype=bool)
        ring[2:-2, 2:-2] = False
        assert np.allclose(qp[:, ring], expect, rtol=0, atol=1e-15)


def test_coarse_interp_is_conservative_r2():
    """R = 2: the 2x2 ghost children of a coarse cell average to its value."""
    o, cd, fd, dxc, dxf = two_level(2, [(6, 6, 4, 4)])
    qc = np.random.default_rng(0).uniform(-1, 1, 3 * 64)
    o.set_level(1, cd, qc)
    o.set_level(2, fd, np.zeros(3 * 16))
    o.fill_ghost(2, 0.0)
    qp = o.read_padded(2, 0)           # fine patch covers coarse cells 3..4
    C = qc.reshape(3, 8, 8)
    # left ghost columns (fine -2,-1 -> fine global 4,5 -> coarse column 2)
    for k in range(2):                  # coarse rows 3, 4
        blk = qp[:, 2 + 2 * k:4 + 2 * k, 0:2]
        assert np.allclose(blk.mean(axis=(1, 2)), C[:, 3 + k, 2], atol=1e-15)


# ---------------------------------------------------------------------------
# Pin of the coarse-interpolation slope (reading R10 of P:131, "interpolated
# from underlying coarse grid patches"): minmod of the two one-sided coarse
# differences, 0 at a coarse local extremum.  The fields are separable, so each
# slope is read off the coarse sequences by hand (below); every value is dyadic,
# so the comparisons are exact.  An unlimited central slope, a `max` in place of
# the `min`, a dropped extremum test or an x/y (or component) mix-up changes at
# least one hand-derived number here.
#
#   a(Ic) = [0, 0, 1, 3, 4, 4.5, 8, 8]     (x sequence, Ic = 0..7)
#   b(Jc) = [0, 0, 2, 2.5, 2, 1, 0, 0]     (y sequence, Jc = 0..7)
#   p = a(Ic) + b(Jc),  u = a(Ic),  v = b(Jc)
#
# Hand-derived minmod slopes (one-sided differences d- = f(k)-f(k-1), d+ = f(k+1)-f(k)):
#   x, Ic=2: d-=1,   d+=2     -> +1      (central would be 1.5, max 2)
#   x, Ic=3: d-=2,   d+=1     -> +1
#   x, Ic=4: d-=1,   d+=0.5   -> +0.5
#   x, Ic=5: d-=0.5, d+=3.5   -> +0.5    (central 2, max 3.5)
#   y, Jc=2: d-=2,   d+=0.5   -> +0.5
#   y, Jc=3: d-=0.5, d+=-0.5  -> 0       (local maximum; central would be 0)
#   y, Jc=4: d-=-0.5, d+=-1   -> -0.5    (central -0.75, max -1)
#   y, Jc=5: d-=-1,  d+=-1    -> -1
SLOPE_X = {2: 1.0, 3: 1.0, 4: 0.5, 5: 0.5}
SLOPE_Y = {2: 0.5, 3: 0.0, 4: -0.5, 5: -1.0}
A_SEQ = [0, 0, 1, 3, 4, 4.5, 8, 8]
B_SEQ = [0, 0, 2, 2.5, 2, 1, 0, 0]


def _minmod_field():
    Jc, Ic = np.mgrid[0:8, 0:8]
    a = np.asarray(A_SEQ, float)[Ic]
    b = np.asarray(B_SEQ, float)[Jc]
    return np.stack([a + b, a, b])


def _hand_value(I, J, R=2):
    """Fine value at fine global (I, J), R = 2: offsets xi, eta = -1/4 or +1/4."""
    Ic, Jc = I // R, J // R
    xi = -0.25 if I % R == 0 else 0.25
    eta = -0.25 if J % R == 0 else 0.25
    sx, sy = SLOPE_X[Ic], SLOPE_Y[Jc]
    a, b = A_SEQ[Ic], B_SEQ[Jc]
    return np.array([a + b + sx * xi + sy * eta, a + sx * xi, b + sy * eta])


def test_coarse_interp_minmod_slope_hand_values():
    """Ghost frame of a fine patch over coarse cells (3..4)^2, R = 2 (fine
    cells 6..9): every ghost cell equals the hand-derived minmod value."""
    o, cd, fd, dxc, dxf = two_level(2, [(6, 6, 4, 4)])
    o.set_level(1, cd, _minmod_field().ravel())
    o.set_level(2, fd, np.zeros(3 * 16))
    o.fill_ghost(2, 0.0)
    qp = o.read_padded(2, 0)
    # spot values written out in full
    assert list(qp[:, 2, 0]) == [3.25, 0.75, 2.5]      # fine (4,6): coarse (2,3), xi=-1/4, eta=-1/4, sy=0
    assert list(qp[:, 4, 1]) == [3.375, 1.25, 2.125]   # fine (5,8): coarse (2,4), xi=+1/4, eta=-1/4, sy=-1/2
    assert list(qp[:, 0, 0]) == [2.625, 0.75, 1.875]   # fine (4,4): corner, coarse (2,2)
    assert list(qp[:, 7, 7]) == [5.375, 4.625, 0.75]   # fine (11,11): coarse (5,5), xi=eta=+1/4, sx=1/2, sy=-1
    n = 0
    for jj in range(8):
        for ii in range(8):
            if 2 <= ii < 6 and 2 <= jj < 6:
                continue
            I, J = 6 + ii - 2, 6 + jj - 2
            assert np.array_equal(qp[:, jj, ii], _hand_value(I, J)), (I, J, qp[:, jj, ii])
            n += 1
    assert n == 48


def test_regrid_interp_minmod_slope_hand_values():
    """The same rule in the regrid interpolation (new fine cells with no old fine
    data, alpha = 1): a new box over coarse cells 2..5 x 2..5."""
    o = oracle.Oracle((0.0, 1.0, 0.0, 1.0), W.EXTRAP, 4, 2)
    o.set_level(1, W.uniform_level(1, 1, 8, 8, (0.0, 1.0, 0.0, 1.0)), _minmod_field().ravel())
    o.regrid(1, [(2, 2, 4, 4)], 2)
    q = o.read(2, 0)
    assert list(q[:, 2, 2]) == [5.25, 2.75, 2.5]       # fine (6,6): coarse (3,3), xi=-1/4, sx=1, sy=0
    for jj in range(8):
        for ii in range(8):
            assert np.array_equal(q[:, jj, ii], _hand_value(4 + ii, 4 + jj))
