"""Brute-force per-cell evaluation of eq. (W) for tiny patches (<= 8x8).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Independent of
claw_oracle.c: written directly in the edge form of eq. (W),

  Q_ij^{n+1} = Q_ij - dt/dx (A+dQ_{i-1/2,j} + A-dQ_{i+1/2,j})
                    - dt/dy (B+dQ_{i,j-1/2} + B-dQ_{i,j+1/2})
                    - dt/dx (F~_{i+1/2,j} - F~_{i-1/2,j})
                    - dt/dy (G~_{i,j+1/2} - G~_{i,j-1/2}),

where every fluctuation, limited wave and transverse term a cell needs is
recomputed from scratch from the raw cell values (no sweep arrays, no
accumulation).  F~ = 1/2 sum |s|(1-|s|dt/dx) W~ plus the transverse parts
coming from the y-Riemann problems of the two cells sharing the edge (P:94,
P:500 "corner transport"); rpn2/rpt2 are the eigen-splittings of A and B of
P:457-466 (linear acoustics).  Ghost cells are made here with numpy padding
(edge = zero-order extrapolation, wrap = periodic), independently of the
oracle's ghost fill.

Variable media (NEXT-4, R20): with a per-cell (rho, K) array every
Riemann problem is re-solved as a 2x2 linear system (numpy.linalg.solve) in
the eigenvectors of the two media involved -- the left-going wave in the
left cell's medium, the right-going one in the right cell's; for the
transverse split, the down-going part in the medium of the cell below, the
up-going part in the medium of the cell above -- instead of the closed forms
the C oracle uses.
"""
from __future__ import annotations

import numpy as np


def _phi(lim: int, r: float) -> float:
    if lim == 0:
        return 1.0
    if lim == 1:
        return max(0.0, min(1.0, r))
    if lim == 2:
        return max(0.0, min(1.0, 2 * r), min(2.0, r))
    if lim == 3:
        return (r + abs(r)) / (1.0 + abs(r))
    if lim == 4:
        return max(0.0, min((1.0 + r) / 2.0, 2.0, 2.0 * r))
    raise ValueError(lim)


class _Cell:
    """Accessor over a padded patch: cell (i, j) in Clawpack 1-based indexing."""

    def __init__(self, qpad):
        self.q = qpad

    def __call__(self, i, j):
        return self.q[:, j + 1, i + 1]


def _eig(ixy, rho, K):
    c = np.sqrt(K / rho)
    Z = rho * c
    mu, mv = (1, 2) if ixy == 1 else (2, 1)
    r1 = np.zeros(3); r1[0] = -Z; r1[mu] = 1.0       # speed -c
    r2 = np.zeros(3); r2[0] = Z; r2[mu] = 1.0        # speed +c
    return c, Z, mu, mv, r1, r2


def riemann(ixy, ql, qr, rho, K):
    """Waves (2,3) and speeds (2) at an interface with left state ql."""
    c, Z, mu, mv, r1, r2 = _eig(ixy, rho, K)
    dq = qr - ql
    # solve dq[0,mu] = a1 r1 + a2 r2 on the (p, normal-velocity) block
    a1 = (-dq[0] + Z * dq[mu]) / (2 * Z)
    a2 = (dq[0] + Z * dq[mu]) / (2 * Z)
    return np.array([a1 * r1, a2 * r2]), np.array([-c, c])


def transverse(ixy, asdq, rho, K):
    """Split asdq (from a sweep in direction ixy) by the eigenvectors of the
    other direction's matrix: returns (down-going part, up-going part)."""
    other = 2 if ixy == 1 else 1
    c, Z, mu, mv, r1, r2 = _eig(other, rho, K)
    b1 = (-asdq[0] + Z * asdq[mu]) / (2 * Z)
    b2 = (asdq[0] + Z * asdq[mu]) / (2 * Z)
    return -c * b1 * r1, c * b2 * r2


def riemann_vc(ixy, ql, qr, medl, medr):
    """Waves and speeds at an interface between media medl, medr = (rho, K):
    dq = a1 r1(left medium) + a2 r2(right medium) on the (p, normal) block."""
    cl, _, mu, _, r1, _ = _eig(ixy, *medl)
    cr, _, _, _, _, r2 = _eig(ixy, *medr)
    dq = qr - ql
    a = np.linalg.solve(np.array([[r1[0], r2[0]], [r1[mu], r2[mu]]]), np.array([dq[0], dq[mu]]))
    return np.array([a[0] * r1, a[1] * r2]), np.array([-cl, cr])


def transverse_vc(ixy, asdq, med_lo, med, med_hi):
    """asdq entering a cell of medium `med`, split by the Riemann problems
    across its low / high edges in the other direction (transmitted parts)."""
    other = 2 if ixy == 1 else 1
    c_lo, _, mu, _, r1_lo, _ = _eig(other, *med_lo)
    _, _, _, _, r1_c, r2_c = _eig(other, *med)
    c_hi, _, _, _, _, r2_hi = _eig(other, *med_hi)
    rhs = np.array([asdq[0], asdq[mu]])
    a_lo = np.linalg.solve(np.array([[r1_lo[0], r2_c[0]], [r1_lo[mu], r2_c[mu]]]), rhs)[0]
    a_hi = np.linalg.solve(np.array([[r1_c[0], r2_hi[0]], [r1_c[mu], r2_hi[mu]]]), rhs)[1]
    return -c_lo * a_lo * r1_lo, c_hi * a_hi * r2_hi


class BruteStep:
    def __init__(self, qpad, dx, dy, dt, rho, K, limiter, order_trans, auxpad=None):
        self.Q = _Cell(qpad)
        self.aux = auxpad            # [2][my+4][mx+4] (rho, K) or None
        self.dx, self.dy, self.dt = dx, dy, dt
        self.rho, self.K = rho, K
        self.lim, self.ot = limiter, order_trans

    def med(self, i, j):
        if self.aux is None:
            return (self.rho, self.K)
        return (float(self.aux[0, j + 1, i + 1]), float(self.aux[1, j + 1, i + 1]))

    def _riemann(self, ixy, i, j):
        ql, qr = self._states(ixy, i, j)
        if self.aux is None:
            return riemann(ixy, ql, qr, self.rho, self.K)
        lo = (i - 1, j) if ixy == 1 else (i, j - 1)
        return riemann_vc(ixy, ql, qr, self.med(*lo), self.med(i, j))

    def _states(self, ixy, i, j):
        """(left, right) states at interface (i,j) of direction ixy: the edge
        between cell (i-1,j) and (i,j) for x, (i,j-1) and (i,j) for y."""
        if ixy == 1:
            return self.Q(i - 1, j), self.Q(i, j)
        return self.Q(i, j - 1), self.Q(i, j)

    def fluct(self, ixy, i, j):
        W, s = self._riemann(ixy, i, j)
        return s[0] * W[0], s[1] * W[1]  # A-dQ, A+dQ

    def limited(self, ixy, i, j):
        W, s = self._riemann(ixy, i, j)
        if self.lim == 0:
            return W, s
        out = W.copy()
        for p in range(2):
            nrm = float(W[p] @ W[p])
            if nrm == 0.0:
                continue
            step = -1 if s[p] > 0 else 1  # upwind neighbour interface
            ii, jj = (i + step, j) if ixy == 1 else (i, j + step)
            Wup, _ = self._riemann(ixy, ii, jj)
            out[p] = _phi(self.lim, float(Wup[p] @ W[p]) / nrm) * W[p]
        return out, s

    def cq(self, ixy, i, j):
        dtdn = self.dt / (self.dx if ixy == 1 else self.dy)
        W, s = self.limited(ixy, i, j)
        return sum(abs(s[p]) * (1 - abs(s[p]) * dtdn) * W[p] for p in range(2))

    def _split_in(self, ixy, i, j):
        """The two fluctuations (possibly corrected) entering cell (i,j) from
        its low and high faces in direction ixy: apdq of the low face and amdq
        of the high face."""
        lo = (i, j)
        hi = (i + 1, j) if ixy == 1 else (i, j + 1)
        am_hi, _ = self.fluct(ixy, *hi)
        _, ap_lo = self.fluct(ixy, *lo)
        if self.ot == 2:
            am_hi = am_hi + self.cq(ixy, *hi)
            ap_lo = ap_lo - self.cq(ixy, *lo)
        return ap_lo, am_hi

    def trans_flux(self, ixy, i, j, side):
        """Transverse flux that the ixy-Riemann problems of cell (i,j) put on
        its low (side=0) or high (side=1) edge in the other direction."""
        if self.ot == 0:
            return np.zeros(3)
        dtdn = self.dt / (self.dx if ixy == 1 else self.dy)
        tot = np.zeros(3)
        for a in self._split_in(ixy, i, j):
            if self.aux is None:
                down, up = transverse(ixy, a, self.rho, self.K)
            else:
                lo, hi = ((i, j - 1), (i, j + 1)) if ixy == 1 else ((i - 1, j), (i + 1, j))
                down, up = transverse_vc(ixy, a, self.med(*lo), self.med(i, j), self.med(*hi))
            tot = tot - 0.5 * dtdn * (down if side == 0 else up)
        return tot

    def Ftilde(self, i, j):
        """F~ on the x-edge between cells (i-1,j) and (i,j)."""
        return (0.5 * self.cq(1, i, j) + self.trans_flux(2, i, j, 0)
                + self.trans_flux(2, i - 1, j, 1))

    def Gtilde(self, i, j):
        """G~ on the y-edge between cells (i,j-1) and (i,j)."""
        return (0.5 * self.cq(2, i, j) + self.trans_flux(1, i, j, 0)
                + self.trans_flux(1, i, j - 1, 1))

    def cell(self, i, j):
        r, s = self.dt / self.dx, self.dt / self.dy
        _, apL = self.fluct(1, i, j)
        amR, _ = self.fluct(1, i + 1, j)
        _, bpB = self.fluct(2, i, j)
        bmT, _ = self.fluct(2, i, j + 1)
        return (self.Q(i, j) - r * (apL + amR) - s * (bpB + bmT)
                - r * (self.Ftilde(i + 1, j) - self.Ftilde(i, j))
                - s * (self.Gtilde(i, j + 1) - self.Gtilde(i, j)))


def pad(q: np.ndarray, bc: str = "edge") -> np.ndarray:
    """[3][my][mx] -> [3][my+4][mx+4] with extrapolation ('edge') or periodic
    ('wrap') ghost cells, both axes."""
    return np.pad(q, ((0, 0), (2, 2), (2, 2)), mode=bc)


def brute_step(q, dx, dy, dt, rho=1.0, K=1.0, limiter=4, order_trans=2, bc="edge", aux=None):
    """One step on a single patch (= the whole domain) of shape [3][my][mx];
    aux: per-cell media [2][my][mx] (rho, K) or None (constant rho, K)."""
    _, my, mx = q.shape
    assert mx <= 16 and my <= 16, "brute force is for tiny patches"
    b = BruteStep(pad(q, bc), dx, dy, dt, rho, K, limiter, order_trans,
                  None if aux is None else pad(aux, bc))
    out = np.empty_like(q)
    for j in range(1, my + 1):
        for i in range(1, mx + 1):
            out[:, j - 1, i - 1] = b.cell(i, j)
    return out
