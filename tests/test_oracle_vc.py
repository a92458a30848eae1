"""Pins of the oracle's variable-coefficient acoustics (NEXT-4; heterogeneous
media P:66; per-system normal / transverse solvers P:433-436; the
acoustics matrices A, B of P:457-466 with rho, K varying per cell; DESIGN.md
R20).  What fixes each part, other than the oracle itself:

* rpn2_vc / rpt2_vc: numpy's eigen-decomposition of each medium's A and B
  (P:457-466), the jump split into the left medium's left-going and the right
  medium's right-going eigenvectors;
* a constant medium given per cell: bitwise the constant-coefficient oracle
  (itself pinned in test_oracle_pins.py / test_oracle_brute.py);
* one step on a Riemann problem at a material interface: the exact cell
  averages of the exact solution (middle state from continuity of p and the
  normal velocity, waves at -c_l and +c_r), for every limiter that vanishes
  at theta = 0;
* long runs: reflection and transmission coefficients R = (Z2-Z1)/(Z1+Z2),
  T = 2 Z2/(Z1+Z2) of a smooth pulse at an interface (x and y), and no
  reflection at all when only the sound speed jumps (Z1 = Z2);
* mirror and transpose symmetry with non-symmetric media;
* brute force: oracle/brute.py's per-cell evaluation, which re-solves every
  Riemann problem as a linear system (no closed forms), on random 4x4 / 3x5
  patches with random per-cell media.
"""
import numpy as np
import pytest

import oracle
from oracle.brute import brute_step
from paper_1808_02638_b200 import workloads as W


def A_mat(rho, K):
    return np.array([[0.0, K, 0.0], [1.0 / rho, 0.0, 0.0], [0.0, 0.0, 0.0]])


def B_mat(rho, K):
    return np.array([[0.0, 0.0, K], [0.0, 0.0, 0.0], [1.0 / rho, 0.0, 0.0]])


def eigvec(M, lam):
    """Eigenvector of M for the eigenvalue closest to lam, scaled so that its
    velocity entry is 1."""
    w, V = np.linalg.eig(M)
    k = int(np.argmin(np.abs(w - lam)))
    assert abs(w[k] - lam) < 1e-12
    v = np.real(V[:, k])
    vel = v[1] if abs(v[1]) > abs(v[2]) else v[2]
    return v / vel


@pytest.mark.parametrize("ixy", [1, 2])
def test_rpn2_vc_is_the_eigen_split_of_each_medium(ixy):
    rng = np.random.default_rng(7 + ixy)
    M = A_mat if ixy == 1 else B_mat
    for _ in range(200):
        ql, qr = rng.uniform(-1, 1, 3), rng.uniform(-1, 1, 3)
        rl, kl, rr, kr = rng.uniform(0.3, 3.0, 4)
        cl, cr = np.sqrt(kl / rl), np.sqrt(kr / rr)
        r1 = eigvec(M(rl, kl), -cl)          # left-going, left medium
        r2 = eigvec(M(rr, kr), cr)           # right-going, right medium
        r0 = np.zeros(3); r0[3 - ixy] = 1.0  # zero-speed wave (transverse velocity)
        a = np.linalg.solve(np.stack([r1, r2, r0], axis=1), qr - ql)
        wave, s, am, ap = oracle.rpn2_vc(ixy, ql, qr, rl, kl, rr, kr)
        np.testing.assert_allclose(s, [-cl, cr], rtol=1e-15)
        np.testing.assert_allclose(wave[0], a[0] * r1, rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(wave[1], a[1] * r2, rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(am, -cl * a[0] * r1, rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(ap, cr * a[1] * r2, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("ixy", [1, 2])
def test_rpt2_vc_transmitted_parts_across_the_transverse_edges(ixy):
    """asdq entering a cell, split as a jump across its low transverse edge
    (down-going wave of the medium below + up-going wave of the cell) and
    across its high edge (down-going of the cell + up-going of the medium
    above); B-asdq = -c_m W_down(m), B+asdq = +c_p W_up(p)."""
    rng = np.random.default_rng(17 + ixy)
    M = B_mat if ixy == 1 else A_mat     # transverse direction's matrix
    for _ in range(200):
        asdq = rng.uniform(-1, 1, 3)
        rm, km, rc, kc, rp, kp = rng.uniform(0.3, 3.0, 6)
        cm, cc, cp = np.sqrt(km / rm), np.sqrt(kc / rc), np.sqrt(kp / rp)
        r0 = np.zeros(3); r0[ixy] = 1.0  # zero-speed wave of the transverse split (normal velocity)
        lo = np.linalg.solve(np.stack([eigvec(M(rm, km), -cm), eigvec(M(rc, kc), cc), r0], 1), asdq)
        hi = np.linalg.solve(np.stack([eigvec(M(rc, kc), -cc), eigvec(M(rp, kp), cp), r0], 1), asdq)
        bm, bp = oracle.rpt2_vc(ixy, asdq, rm, km, rc, kc, rp, kp)
        np.testing.assert_allclose(bm, -cm * lo[0] * eigvec(M(rm, km), -cm), rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(bp, cp * hi[1] * eigvec(M(rp, kp), cp), rtol=1e-12, atol=1e-14)


def run(descs, q0, aux, nsteps, dt, limiter=4, order_trans=2, bc=W.EXTRAP, domain=None):
    if domain is None:   # the bounding box of the level
        domain = (float((descs["xlower"]).min()), float((descs["xlower"] + descs["mx"] * descs["dx"]).max()),
                  float((descs["ylower"]).min()), float((descs["ylower"] + descs["my"] * descs["dy"]).max()))
    o = oracle.Oracle(domain, bc, limiter, order_trans, nthreads=2)
    o.set_level(1, descs, q0)
    if aux is not None:
        o.set_aux(1, aux)
    cfl = []
    for n in range(nsteps):
        o.fill_ghost(1, n * dt)
        cfl.append(o.advance_level(1, dt))
    return o.read_level(1), cfl


@pytest.mark.parametrize("limiter", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("order_trans", [0, 1, 2])
def test_constant_medium_per_cell_is_bitwise_the_constant_oracle(limiter, order_trans):
    descs = W.ragged_level(5, 24, 20, 9)
    rho, K = 2.5, 0.7
    descs["rho"], descs["K"] = rho, K
    q0 = W.random_ic(descs, 3)
    aux = np.concatenate([np.concatenate([np.full(int(d["mx"] * d["my"]), rho),
                                          np.full(int(d["mx"] * d["my"]), K)]) for d in descs])
    dt = 0.8 * float(descs["dx"][0]) / np.sqrt(K / rho)
    for bc in (W.EXTRAP, W.PERIODIC):
        a, ca = run(descs, q0, aux, 4, dt, limiter, order_trans, bc)
        b, cb = run(descs, q0, None, 4, dt, limiter, order_trans, bc)
        assert np.array_equal(a, b)
        assert ca == cb


def riemann_exact_step(pL, uL, pR, uR, m1, m2, nu1, nu2):
    """Exact cell averages after one step of the Riemann problem at a
    material interface (textbook: continuity of p and of the normal velocity
    across the interface; left-going wave at -c1 in medium 1, right-going at
    +c2 in medium 2): the cell left of the interface becomes
    (1-nu1) qL + nu1 qm, the one right of it (1-nu2) qR + nu2 qm."""
    Z1 = m1[0] * np.sqrt(m1[1] / m1[0])
    Z2 = m2[0] * np.sqrt(m2[1] / m2[0])
    um = (pL - pR + Z1 * uL + Z2 * uR) / (Z1 + Z2)
    pm = (Z2 * pL + Z1 * pR + Z1 * Z2 * (uL - uR)) / (Z1 + Z2)
    return ((1 - nu1) * pL + nu1 * pm, (1 - nu1) * uL + nu1 * um,
            (1 - nu2) * pR + nu2 * pm, (1 - nu2) * uR + nu2 * um)


@pytest.mark.parametrize("limiter", [1, 2, 3, 4])
@pytest.mark.parametrize("axis", ["x", "y"])
@pytest.mark.parametrize("media", [((1.0, 1.0), (4.0, 1.0)), ((2.0, 0.5), (0.5, 2.0)),
                                   ((1.0, 4.0), (0.25, 1.0))])
def test_one_step_at_a_material_interface_is_the_exact_riemann_solution(limiter, axis, media):
    n, w = 16, 3
    m1, m2 = media
    dx = 2.0 / n
    c1, c2 = np.sqrt(m1[1] / m1[0]), np.sqrt(m2[1] / m2[0])
    dt = 0.8 * dx / max(c1, c2)
    pL, uL, vL, pR, uR, vR = 0.7, -0.3, 0.2, -0.4, 0.5, -0.6
    if axis == "x":
        descs = W.uniform_level(1, 1, n, w, (-1.0, 1.0, 0.0, w * dx))
        sel = lambda a: a[:, :, : n // 2]          # noqa: E731  left half (x < 0)
        shape = (w, n)
    else:
        descs = W.uniform_level(1, 1, w, n, (0.0, w * dx, -1.0, 1.0))
        sel = lambda a: a[:, : n // 2, :]          # noqa: E731
        shape = (n, w)
    q = np.zeros((3,) + shape)
    aux = np.zeros((2,) + shape)
    nrm, tan = (1, 2) if axis == "x" else (2, 1)
    q[0], q[nrm], q[tan] = pR, uR, vR
    aux[0], aux[1] = m2
    sel(q)[0], sel(q)[nrm], sel(q)[tan] = pL, uL, vL
    sel(aux)[0], sel(aux)[1] = m1
    out, cfl = run(descs, q.ravel(), aux.ravel(), 1, dt, limiter, 2)
    out = out.reshape(q.shape)
    pl, ul, pr, ur = riemann_exact_step(pL, uL, pR, uR, m1, m2, c1 * dt / dx, c2 * dt / dx)
    exp = q.copy()
    if axis == "x":
        exp[0][:, n // 2 - 1], exp[nrm][:, n // 2 - 1] = pl, ul
        exp[0][:, n // 2], exp[nrm][:, n // 2] = pr, ur
    else:
        exp[0][n // 2 - 1, :], exp[nrm][n // 2 - 1, :] = pl, ul
        exp[0][n // 2, :], exp[nrm][n // 2, :] = pr, ur
    np.testing.assert_allclose(out, exp, rtol=0, atol=2e-15)
    assert cfl[0] == pytest.approx(max(c1, c2) * dt / dx, rel=1e-15)


def pulse_run(Z1c1, Z2c2, axis, n=480, w=2, steps=None, limiter=4):
    """Right-going smooth pressure pulse in medium 1 (x < 0) hits medium 2."""
    (Z1, c1), (Z2, c2) = Z1c1, Z2c2
    m1, m2 = (Z1 / c1, Z1 * c1), (Z2 / c2, Z2 * c2)     # rho = Z/c, K = Z c
    dx = 2.0 / n
    xc = -1.0 + (np.arange(n) + 0.5) * dx
    p = np.where(np.abs(xc + 0.5) < 0.2, np.cos(np.pi * (xc + 0.5) / 0.4) ** 2, 0.0)
    q = np.zeros((3, w, n))
    q[0] = p
    q[1] = p / Z1
    aux = np.zeros((2, w, n))
    aux[0], aux[1] = np.where(xc < 0, m1[0], m2[0]), np.where(xc < 0, m1[1], m2[1])
    descs = W.uniform_level(1, 1, n, w, (-1.0, 1.0, 0.0, w * dx))
    if axis == "y":
        q = np.stack([q[0].T, q[2].T, q[1].T])
        aux = np.stack([aux[0].T, aux[1].T])
        descs = W.uniform_level(1, 1, w, n, (0.0, w * dx, -1.0, 1.0))
    dt = 0.9 * dx / max(c1, c2)
    # the incident pulse [-0.7, -0.3] has fully reached the interface at
    # t = 0.7 / c1; run until both its parts are 0.1 away from it
    t_end = 0.7 / c1 + 0.1 / min(c1, c2)
    steps = steps or int(np.ceil(t_end / dt))
    out, _ = run(descs, q.ravel(), aux.ravel(), steps, dt, limiter, 2)
    out = out.reshape(q.shape)
    pp = out[0] if axis == "x" else out[0].T
    return xc, pp


@pytest.mark.parametrize("axis", ["x", "y"])
@pytest.mark.parametrize("Z2c2", [(3.0, 1.0), (1.0 / 3.0, 2.0), (2.0, 0.5)])
def test_reflection_and_transmission_coefficients(axis, Z2c2):
    Z1, c1 = 1.0, 1.0
    Z2, c2 = Z2c2
    xc, p = pulse_run((Z1, c1), (Z2, c2), axis)
    R = (Z2 - Z1) / (Z1 + Z2)
    T = 2 * Z2 / (Z1 + Z2)
    left, right = p[:, xc < -0.05], p[:, xc > 0.05]
    # incident amplitude 1; the extreme of each separated pulse
    refl = left.flat[np.argmax(np.abs(left))]
    trans = right.flat[np.argmax(np.abs(right))]
    assert abs(refl - R) < 0.02, (refl, R)
    assert abs(trans - T) < 0.02, (trans, T)
    assert np.array_equal(p[0], p[-1])   # y-independent (transverse terms cancel)


def test_matched_impedance_reflects_nothing():
    """Z1 = Z2 with c2 = 2 c1: the incident wave passes the speed jump with
    no reflected wave (alpha_1 = 0 at every interface), to rounding."""
    xc, p = pulse_run((1.0, 1.0), (1.0, 2.0), "x")
    assert np.abs(p[:, xc < -0.05]).max() < 1e-13
    assert np.abs(p[:, xc > 0.05]).max() > 0.9


def random_case(seed, mx, my):
    rng = np.random.default_rng(seed)
    q = rng.uniform(-1, 1, (3, my, mx))
    aux = rng.uniform(0.4, 2.5, (2, my, mx))
    return q, aux


@pytest.mark.parametrize("order_trans", [0, 1, 2])
def test_mirror_and_transpose_symmetry(order_trans):
    mx = my = 12
    q, aux = random_case(50 + order_trans, mx, my)
    dx = 2.0 / mx
    cmax = np.sqrt(aux[1] / aux[0]).max()
    dt = 0.7 * dx / cmax
    descs = W.uniform_level(1, 1, mx, my)

    def go(qq, aa):
        return run(descs, qq.ravel(), aa.ravel(), 3, dt, 4, order_trans)[0].reshape(3, my, mx)

    base = go(q, aux)
    # mirror x: p(x) -> p(-x), u -> -u
    qm = q[:, :, ::-1].copy(); qm[1] *= -1
    got = go(qm, aux[:, :, ::-1].copy())
    exp = base[:, :, ::-1].copy(); exp[1] *= -1
    assert np.abs(got - exp).max() <= 1e-13
    # transpose: x <-> y, u <-> v
    qt = np.stack([q[0].T, q[2].T, q[1].T]).copy()
    got = go(qt, np.stack([aux[0].T, aux[1].T]).copy())
    exp = np.stack([base[0].T, base[2].T, base[1].T])
    assert np.abs(got - exp).max() <= 1e-13


@pytest.mark.parametrize("limiter", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("order_trans", [0, 1, 2])
@pytest.mark.parametrize("shape,nsteps", [((4, 4), 1), ((4, 4), 3), ((3, 5), 2)])
def test_vc_oracle_equals_brute_force(limiter, order_trans, shape, nsteps):
    my, mx = shape
    seed = 1000 + 100 * limiter + 10 * order_trans + nsteps
    q, aux = random_case(seed, mx, my)
    dx, dy = 0.5, 0.4
    cmax = np.sqrt(aux[1] / aux[0]).max()
    dt = (0.8 if order_trans else 0.4) * min(dx, dy) / cmax
    bc, mode = (W.EXTRAP, "edge") if seed % 2 else (W.PERIODIC, "wrap")
    dom = (0.0, mx * dx, 0.0, my * dy)
    descs = W.make_descs([0], [0], mx, my, dx, dy, dom)
    got, _ = run(descs, q.ravel(), aux.ravel(), nsteps, dt, limiter, order_trans, bc, dom)
    ref = q.copy()
    for _ in range(nsteps):
        ref = brute_step(ref, dx, dy, dt, limiter=limiter, order_trans=order_trans, bc=mode, aux=aux)
    assert np.abs(got.reshape(ref.shape) - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max())


def test_vc_cfl_is_the_per_face_maximum():
    """Courant number = max over swept faces of |s| dt/dx with s = -c_l, +c_r
    (P:230-232): the fastest cell's c, including faces of ghost rows."""
    descs = W.ragged_level(2, 20, 16, 8)
    aux = W.random_media(descs, 4)
    dt = 0.01
    _, cfl = run(descs, W.random_ic(descs, 4), aux, 1, dt)
    cmax = W.max_sound_speed(aux, descs)
    assert cfl[0] == pytest.approx(cmax * dt / float(descs["dx"][0]), rel=1e-15)


def test_vc_tiling_invariance_bitwise():
    """A medium and state on one 24x20 patch = the same on a ragged tiling."""
    big = W.uniform_level(1, 1, 24, 20)
    tiled = W.ragged_level(9, 24, 20, 7)
    rng = np.random.default_rng(3)
    Q = rng.uniform(-1, 1, (3, 20, 24))
    A = rng.uniform(0.5, 2.0, (2, 20, 24))

    def split(F, descs, m):
        out = []
        for d in descs:
            i0 = int(round((d["xlower"] + 1) / d["dx"])); j0 = int(round((d["ylower"] + 1) / d["dy"]))
            out.append(F[:, j0:j0 + d["my"], i0:i0 + d["mx"]].ravel())
        return np.concatenate(out)

    dt = 0.5 * float(big["dx"][0])
    a, _ = run(big, Q.ravel(), A.ravel(), 3, dt)
    b, _ = run(tiled, split(Q, tiled, 3), split(A, tiled, 2), 3, dt)
    assert np.array_equal(split(a.reshape(3, 20, 24), tiled, 3), b)


def test_set_aux_errors():
    descs = W.uniform_level(2, 1, 4, 4)
    o = oracle.Oracle(W.DOMAIN, W.EXTRAP, 4, 2)
    o.set_level(1, descs, None)
    bad = np.ones(2 * 32); bad[5] = 0.0
    with pytest.raises(oracle.OracleError):
        o.set_aux(1, bad)
    o.set_aux(1, np.ones(64))
    with pytest.raises(oracle.OracleError):   # single-level only (R20)
        o.set_level(2, W.make_descs([0], [0], 4, 4, 0.25, 0.5), None)
