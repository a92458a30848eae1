"""Oracle (sweep-structured C) vs brute force (per-cell NumPy evaluation of
eq. (W)) on tiny patches (S:170 idea: 4x4 at 1e-13)."""
import numpy as np
import pytest

import oracle
from oracle.brute import brute_step
from paper_1808_02638_b200 import workloads as W


def oracle_steps(q, dx, dy, dt, nsteps, limiter, order_trans, bc, rho=1.0, K=1.0):
    _, my, mx = q.shape
    dom = (0.0, mx * dx, 0.0, my * dy)
    o = oracle.Oracle(dom, bc, limiter, order_trans, nthreads=1)
    o.set_level(1, W.make_descs([0], [0], mx, my, dx, dy, dom, rho, K), q.ravel())
    for n in range(nsteps):
        o.fill_ghost(1, n * dt)
        o.advance_level(1, dt)
    return o.read(1, 0)


@pytest.mark.parametrize("limiter", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("order_trans", [0, 1, 2])
@pytest.mark.parametrize("shape,nsteps", [((4, 4), 1), ((4, 4), 5), ((3, 5), 3)])
def test_oracle_equals_brute_force(limiter, order_trans, shape, nsteps):
    my, mx = shape
    seed = 100 * limiter + 10 * order_trans + nsteps
    rng = np.random.default_rng(seed)
    q = rng.uniform(-1, 1, (3, my, mx))
    rho, K = rng.uniform(0.5, 2.0, 2)
    dx, dy = 0.5, 0.4
    c = np.sqrt(K / rho)
    dt = (0.8 if order_trans else 0.4) * min(dx, dy) / c
    bc, mode = (W.EXTRAP, "edge") if seed % 2 else (W.PERIODIC, "wrap")
    got = oracle_steps(q, dx, dy, dt, nsteps, limiter, order_trans, bc, rho, K)
    ref = q.copy()
    for _ in range(nsteps):
        ref = brute_step(ref, dx, dy, dt, rho, K, limiter, order_trans, bc=mode)
    assert np.abs(got - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max())
