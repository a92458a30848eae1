"""Pins of the CPU oracle against what the paper and the mathematics fix.

Each test names the passage it pins (P:a-b = PAPER.md lines, S:a-b = SPEC.md
lines; SPEC worked examples are used as test ideas only).  None of these
re-types the oracle's formulas: they use the paper's matrices and
numpy's eigen-decomposition, closed-form solutions (Lax-Wendroff, exact
translation, plane waves), invariants (conservation, symmetry, tiling) and
hand-derived dyadic examples.
"""
import math

import numpy as np
import pytest

import oracle
from paper_1808_02638_b200 import workloads as W


def paper_A(rho, K):
    """A of P:457-461 (flux Jacobian in x)."""
    return np.array([[0.0, K, 0.0], [1.0 / rho, 0.0, 0.0], [0.0, 0.0, 0.0]])


def paper_B(rho, K):
    """B of P:462-466 (flux Jacobian in y)."""
    return np.array([[0.0, 0.0, K], [0.0, 0.0, 0.0], [1.0 / rho, 0.0, 0.0]])


def split(M):
    """M^- and M^+ from numpy's eigen-decomposition (independent of rpn2)."""
    lam, R = np.linalg.eig(M)
    lam = lam.real
    R = R.real
    Ri = np.linalg.inv(R)
    return R @ np.diag(np.minimum(lam, 0)) @ Ri, R @ np.diag(np.maximum(lam, 0)) @ Ri


# --------------------------------------------------------------------------
# Riemann solvers
# --------------------------------------------------------------------------

def test_rpn2_worked_example():
    # ql = (1,0,0), qr = 0, rho = K = 1
    wave, s, am, ap = oracle.rpn2(1, [1, 0, 0], [0, 0, 0])
    assert np.array_equal(am, [0.5, -0.5, 0.0])
    assert np.array_equal(ap, [-0.5, -0.5, 0.0])
    assert np.array_equal(s, [-1.0, 1.0])
    # zero jump -> zero waves
    wave, s, am, ap = oracle.rpn2(2, [0.3, -2, 5], [0.3, -2, 5])
    assert not wave.any() and not am.any() and not ap.any()


@pytest.mark.parametrize("ixy", [1, 2])
def test_rpn2_matches_eigensplit_of_paper_matrix(ixy):
    rng = np.random.default_rng(11 + ixy)
    for _ in range(2000):
        rho, K = rng.uniform(0.2, 5.0, 2)
        ql, qr = rng.uniform(-3, 3, 3), rng.uniform(-3, 3, 3)
        M = paper_A(rho, K) if ixy == 1 else paper_B(rho, K)
        Mm, Mp = split(M)
        wave, s, am, ap = oracle.rpn2(ixy, ql, qr, rho, K)
        dq = qr - ql
        scale = 1e-13 * max(1.0, np.abs(M).max() * np.abs(dq).max())
        assert np.abs(am + ap - M @ dq).max() <= scale        # S:543 consistency
        assert np.abs(am - Mm @ dq).max() <= scale
        assert np.abs(ap - Mp @ dq).max() <= scale
        c = math.sqrt(K / rho)
        assert np.allclose(s, [-c, c], rtol=1e-15, atol=0)
        assert np.abs(wave.sum(axis=0)[[0, ixy]] - dq[[0, ixy]]).max() <= scale


@pytest.mark.parametrize("ixy", [1, 2])
def test_rpt2_matches_transverse_eigensplit(ixy):
    # S:117 worked example
    bm, bp = oracle.rpt2(1, [1, 0, 0])
    assert np.array_equal(bm, [-0.5, 0.0, 0.5]) and np.array_equal(bp, [0.5, 0.0, 0.5])
    rng = np.random.default_rng(5 + ixy)
    for _ in range(2000):
        rho, K = rng.uniform(0.2, 5.0, 2)
        asdq = rng.uniform(-3, 3, 3)
        T = paper_B(rho, K) if ixy == 1 else paper_A(rho, K)   # transverse matrix
        Tm, Tp = split(T)
        bm, bp = oracle.rpt2(ixy, asdq, rho, K)
        scale = 1e-13 * max(1.0, np.abs(T).max() * np.abs(asdq).max())
        assert np.abs(bm + bp - T @ asdq).max() <= scale
        assert np.abs(bm - Tm @ asdq).max() <= scale
        assert np.abs(bp - Tp @ asdq).max() <= scale


# --------------------------------------------------------------------------
# Limiter phi(theta) (Clawpack numbering)
# --------------------------------------------------------------------------

THETAS = [-1.0, 0.0, 0.25, 1 / 3, 0.5, 1.0, 2.0, 3.0, 10.0]


def test_philim_values():
    mc = [0, 0, 0.5, 2 / 3, 0.75, 1, 1.5, 2, 2]
    mm = [0, 0, 0.25, 1 / 3, 0.5, 1, 1, 1, 1]
    sb = [0, 0, 0.5, 2 / 3, 1, 1, 2, 2, 2]
    for th, a, b, c in zip(THETAS, mc, mm, sb):
        assert oracle.philim(4, th) == pytest.approx(a, abs=1e-16)
        assert oracle.philim(1, th) == pytest.approx(b, abs=1e-16)
        assert oracle.philim(2, th) == pytest.approx(c, abs=1e-16)
        assert oracle.philim(0, th) == 1.0
    assert oracle.philim(3, 3.0) == 1.5          # S:127 van Leer
    assert oracle.philim(3, -2.0) == 0.0
    assert oracle.philim(3, 1.0) == 1.0


# --------------------------------------------------------------------------
# helpers
# --------------------------------------------------------------------------

def single_patch(q, dx=1.0, dy=1.0, bc=W.EXTRAP, limiter=4, order_trans=2, rho=1.0, K=1.0):
    _, my, mx = q.shape
    o = oracle.Oracle((0.0, mx * dx, 0.0, my * dy), bc, limiter, order_trans, nthreads=1)
    d = W.make_descs([0], [0], mx, my, dx, dy, (0.0, mx * dx, 0.0, my * dy), rho, K)
    o.set_level(1, d, q.ravel())
    return o


def run(o, nsteps, dt, level=1):
    c = 0.0
    for n in range(nsteps):
        o.fill_ghost(level, n * dt)
        c = o.advance_level(level, dt)
    return c


# --------------------------------------------------------------------------
# Hand-derived one-step examples (every intermediate dyadic => bitwise)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("limiter", [0, 1, 2, 3, 4])
def test_hand_example_1d_step(limiter):
    q = np.zeros((3, 4, 4))
    q[0, :, :2] = 1.0                      # p = 1 for i <= 2 (1-based)
    o = single_patch(q, limiter=limiter)
    cfl = run(o, 1, 0.5)
    out = o.read(1, 0)
    if limiter == 0:
        p_row = [1.0, 0.875, 0.125, 0.0]
    else:
        p_row = [1.0, 0.75, 0.25, 0.0]
    for j in range(4):
        assert np.array_equal(out[0, j], p_row)
        assert np.array_equal(out[1, j], [0.0, 0.25, 0.25, 0.0])
        assert not out[2, j].any()
    assert cfl == 0.5


def spike_expected(kind):
    p = np.zeros((5, 5)); u = np.zeros((5, 5)); v = np.zeros((5, 5))  # [i][j], 0-based
    if kind == "mc":
        p[1:4, 1:4] = np.array([[1, 2, 1], [2, 4, 2], [1, 2, 1]]) / 16.0
        u[1, 1:4] = [-1 / 32, -3 / 16, -1 / 32]
        u[3, 1:4] = [1 / 32, 3 / 16, 1 / 32]
        v[1:4, 1] = [-1 / 32, -3 / 16, -1 / 32]
        v[1:4, 3] = [1 / 32, 3 / 16, 1 / 32]
    else:
        p[2, 2] = 0.5
        p[1, 2] = p[3, 2] = p[2, 1] = p[2, 3] = 0.125
        u[1, 2], u[3, 2] = -0.25, 0.25
        v[2, 1], v[2, 3] = -0.25, 0.25
    return p, u, v


@pytest.mark.parametrize("limiter,order_trans,kind", [(4, 2, "mc"), (4, 1, "mc"), (0, 2, "lw")])
def test_hand_example_2d_spike(limiter, order_trans, kind):
    """Corner transport pin: a pressure spike, one step at nu = 1/2."""
    q = np.zeros((3, 5, 5))
    q[0, 2, 2] = 1.0
    o = single_patch(q, limiter=limiter, order_trans=order_trans)
    run(o, 1, 0.5)
    out = o.read(1, 0)                    # [m][j][i]
    p, u, v = spike_expected(kind)        # [i][j]
    assert np.array_equal(out[0].T, p)
    assert np.array_equal(out[1].T, u)
    assert np.array_equal(out[2].T, v)
    assert out[0].sum() == 1.0 and out[1].sum() == 0.0 and out[2].sum() == 0.0


# --------------------------------------------------------------------------
# Closed forms
# --------------------------------------------------------------------------

@pytest.mark.parametrize("rho,K", [(1.0, 1.0), (2.0, 0.5), (0.7, 3.1)])
def test_limiter_off_equals_1d_lax_wendroff(rho, K):
    """Limiter off, y-independent data: the method reduces to 1D Lax-Wendroff
    Q - r/2 A (Q+ - Q-) + r^2/2 A^2 (Q+ - 2Q + Q-) with A of P:457-461."""
    rng = np.random.default_rng(3)
    mx, my = 12, 4
    row = rng.uniform(-1, 1, (3, mx))
    q = np.repeat(row[:, None, :], my, axis=1)
    c = math.sqrt(K / rho)
    dx = 0.1
    dt = 0.7 * dx / c
    o = single_patch(q, dx=dx, dy=dx, bc=W.PERIODIC, limiter=0, rho=rho, K=K)
    run(o, 1, dt)
    out = o.read(1, 0)
    A = paper_A(rho, K)
    r = dt / dx
    qp, qm = np.roll(row, -1, axis=1), np.roll(row, 1, axis=1)
    lw = row - 0.5 * r * A @ (qp - qm) + 0.5 * r * r * (A @ A) @ (qp - 2 * row + qm)
    for j in range(my):
        assert np.abs(out[:, j, :] - lw).max() <= 1e-14 * max(1.0, np.abs(row).max())


def test_cfl_one_translation():
    """Right-going plane wave p = Z u, nu = 1, periodic: exact one-cell shift
    per step (P:230-232 with nu = 1); after mx steps q = q0."""
    mx, my = 24, 3
    x = (np.arange(mx) + 0.5) / mx
    prof = np.sin(2 * np.pi * x) + 0.3 * np.cos(6 * np.pi * x)
    q = np.zeros((3, my, mx))
    q[0] = prof
    q[1] = prof                            # Z = 1
    for limiter in (0, 4):
        o = single_patch(q, dx=1.0 / mx, dy=1.0 / mx, bc=W.PERIODIC, limiter=limiter)
        dt = 1.0 / mx
        for n in range(mx):
            o.fill_ghost(1, n * dt)
            cfl = o.advance_level(1, dt)
            out = o.read(1, 0)
            assert np.abs(out[0] - np.roll(q[0], n + 1, axis=1)).max() <= 1e-15
            assert np.abs(out[1] - np.roll(q[1], n + 1, axis=1)).max() <= 1e-15
            assert np.abs(out[2]).max() <= 1e-15
        assert cfl == 1.0


@pytest.mark.parametrize("limiter", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("order_trans", [0, 1, 2])
def test_conservation_periodic(limiter, order_trans):
    """Flux-difference form telescopes: with periodic BCs sum(p), sum(u),
    sum(v) are constant (eq. (W))."""
    rng = np.random.default_rng(limiter * 7 + order_trans)
    q = rng.uniform(-1, 1, (3, 16, 16))
    o = single_patch(q, dx=1 / 16, dy=1 / 16, bc=W.PERIODIC, limiter=limiter,
                     order_trans=order_trans)
    s0 = q.sum(axis=(1, 2))
    # without transverse terms the unsplit scheme is only stable for nu <= 1/2
    run(o, 20, (0.9 if order_trans else 0.45) / 16)
    q1 = o.read(1, 0)
    s1 = q1.sum(axis=(1, 2))
    assert np.abs(q1).max() < 10.0
    assert np.abs(s1 - s0).max() <= 1e-14 * np.abs(q).sum()


def comp_sums(flat, descs):
    offs = W.level_offsets(descs)
    tot = np.zeros(3)
    for p, d in enumerate(descs):
        tot += flat[offs[p]:offs[p + 1]].reshape(3, -1).sum(axis=1)
    return tot


def rebox(base, domain):
    """Re-place a ragged level's integer boxes on another domain."""
    i0 = np.rint((base["xlower"] + 1) / base["dx"]).astype(int)
    j0 = np.rint((base["ylower"] + 1) / base["dy"]).astype(int)
    nx = int(round(2 / base["dx"][0])); ny = int(round(2 / base["dy"][0]))
    dx = (domain[1] - domain[0]) / nx; dy = (domain[3] - domain[2]) / ny
    return np.concatenate([W.make_descs([a], [b], int(m), int(n), dx, dy, domain)
                           for a, b, m, n in zip(i0, j0, base["mx"], base["my"])]), i0, j0


def test_conservation_tiled_periodic_level():
    d, _, _ = rebox(W.ragged_level(4, 24, 20, 9), (0, 1, 0, 1))
    q0 = W.random_ic(d, 9)
    o = oracle.Oracle((0, 1, 0, 1), W.PERIODIC, 4, 2, nthreads=2)
    o.set_level(1, d, q0)
    run(o, 10, 0.8 / 24)
    s0, s1 = comp_sums(q0, d), comp_sums(o.read_level(1), d)
    assert np.abs(s1 - s0).max() <= 1e-13 * np.abs(q0).sum()


def test_radial_symmetry():
    """Ring centred on a square patch: p(i,j) = p(j,i), u(i,j) = v(j,i);
    mirror in x: p even, u odd (P:469-471 benchmark is radially symmetric)."""
    d = W.uniform_level(1, 1, 40, 40)
    q0 = W.ring_ic(d)
    o = oracle.Oracle(W.DOMAIN, W.EXTRAP, 4, 2, nthreads=1)
    o.set_level(1, d, q0)
    run(o, 10, 0.9 * 2 / 40)
    q = o.read(1, 0)
    tol = 1e-15 * np.abs(q).max() * 4
    assert np.abs(q[0] - q[0].T).max() <= tol
    assert np.abs(q[1] - q[2].T).max() <= tol
    assert np.abs(q[0] - q[0][:, ::-1]).max() <= tol
    assert np.abs(q[1] + q[1][:, ::-1]).max() <= tol
    assert np.abs(q[2] - q[2][:, ::-1]).max() <= tol
    assert np.abs(q[0]).max() > 0.1


@pytest.mark.parametrize("limiter", [1, 4])
def test_tiling_invariance_bitwise(limiter):
    """A level split into patches gives bitwise the same result as one patch
    (ghost copies are exact; each interface's arithmetic is unchanged)."""
    n = 24
    big = W.uniform_level(1, 1, n, n)
    q0 = W.random_ic(big, 1)
    o1 = oracle.Oracle(W.DOMAIN, W.EXTRAP, limiter, 2, nthreads=1)
    o1.set_level(1, big, q0)
    run(o1, 5, 0.8 * 2 / n)
    ref = o1.read(1, 0)
    base = W.ragged_level(2, n, n, 7)
    full = q0.reshape(3, n, n)
    base, i0, j0 = rebox(base, W.DOMAIN)
    parts = [full[:, b:b + h, a:a + w].ravel() for a, b, w, h in
             zip(i0, j0, base["mx"], base["my"])]
    o2 = oracle.Oracle(W.DOMAIN, W.EXTRAP, limiter, 2, nthreads=3)
    o2.set_level(1, base, np.concatenate(parts))
    run(o2, 5, 0.8 * 2 / n)
    for p, (a, b, w, h) in enumerate(zip(i0, j0, base["mx"], base["my"])):
        assert np.array_equal(o2.read(1, p), ref[:, b:b + h, a:a + w])


def _plane_wave_error(N, limiter):
    h = 1.0 / N
    T = 0.25
    nsteps = int(math.ceil(T / (0.8 * h)))
    dt = T / nsteps
    xc = (np.arange(N) + 0.5) * h
    X, Y = np.meshgrid(xc, xc)
    f = (math.sin(math.pi * h) / (math.pi * h)) ** 2     # exact cell average factor
    k = 2 * math.pi
    def avg(t):
        return f * np.sin(k * (X + Y - math.sqrt(2) * t))
    q = np.stack([avg(0), avg(0) / math.sqrt(2), avg(0) / math.sqrt(2)])
    o = single_patch(q, dx=h, dy=h, bc=W.PERIODIC, limiter=limiter)
    run(o, nsteps, dt)
    return np.abs(o.read(1, 0)[0] - avg(T)).mean()


@pytest.mark.parametrize("limiter", [0])
def test_second_order_convergence(limiter):
    """Second order on smooth data ('high-resolution'): the L1 error
    ratio per grid doubling is >= 3.5 with the limiter off."""
    e = [_plane_wave_error(N, limiter) for N in (16, 32, 64)]
    assert e[0] / e[1] >= 3.5 and e[1] / e[2] >= 3.5, e


def test_mc_converges():
    e = [_plane_wave_error(N, 4) for N in (16, 32, 64)]
    assert e[0] / e[1] >= 3.0 and e[1] / e[2] >= 3.0, e


def test_trivial_cases():
    rng = np.random.default_rng(0)
    const = np.ones((3, 6, 7)) * np.array([0.3, -1.2, 2.5])[:, None, None]
    o = single_patch(const)
    run(o, 3, 0.4)
    assert np.array_equal(o.read(1, 0), const)            # constant state
    q = rng.uniform(-1, 1, (3, 6, 7))
    o = single_patch(q)
    cfl = run(o, 1, 0.0)
    assert cfl == 0.0 and np.array_equal(o.read(1, 0), q)  # dt = 0


def test_linearity_limiter_off():
    rng = np.random.default_rng(1)
    a, b = rng.uniform(-1, 1, (2, 3, 8, 8))
    outs = []
    for q in (a, b, 2.0 * a - 3.0 * b):
        o = single_patch(q, limiter=0, bc=W.PERIODIC)
        run(o, 2, 0.4)
        outs.append(o.read(1, 0))
    assert np.abs(outs[2] - (2 * outs[0] - 3 * outs[1])).max() <= 1e-13


def test_cfl_value_closed_form():
    """cfl = c dt / min(dx, dy) (max over both sweeps)."""
    rho, K = 1.7, 0.6
    q = np.random.default_rng(2).uniform(-1, 1, (3, 5, 9))
    o = single_patch(q, dx=0.1, dy=0.05, rho=rho, K=K)
    dt = 0.013
    cfl = run(o, 1, dt)
    c = math.sqrt(K / rho)
    assert cfl == max((dt / 0.1) * c, (dt / 0.05) * c)


def test_level_cfl_is_max_of_patches():
    d = W.ragged_level(5, 20, 16, 8)
    o = oracle.Oracle(W.DOMAIN, W.EXTRAP, 4, 2, nthreads=2)
    o.set_level(1, d, W.random_ic(d, 0))
    o.fill_ghost(1)
    c = o.advance_level(1, 0.05)
    pc = [o.patch_cfl(1, p) for p in range(len(d))]
    assert c == max(pc)
