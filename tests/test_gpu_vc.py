"""GPU parity of variable-coefficient acoustics (NEXT-4: per-cell rho, K,
P:66; R20): libclaw's step_vc_kernel through the
C-ABI (claw_set_aux) against the oracle's vc step (tests/test_oracle_vc.py pins
it) on the same seeded inputs.

Bar (BASELINE.json north_star): max|q_gpu - q_oracle| <= 1e-12 max|q_oracle|
(after 100 steps where stated); the CFL -- here a genuine per-face maximum of
max(c_l, c_r) dt/dx over every swept face -- bitwise equal to the oracle's.
"""
import os

import numpy as np
import pytest

import oracle
from paper_1808_02638_b200 import binding, workloads as W

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    binding.load()


def rel_err(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def pair(descs, q0, aux, limiter=4, ot=2, bc=W.EXTRAP, domain=W.DOMAIN):
    g = binding.Claw(domain, bc, limiter, ot, device=0)
    g.set_level(1, descs, q0)
    assert g.level_mode(1) == "grid"
    g.set_aux(1, aux)
    o = oracle.Oracle(domain, bc, limiter, ot, nthreads=0)
    o.set_level(1, descs, q0)
    o.set_aux(1, aux)
    return g, o


def run(g, o, nsteps, dt, check_every=0):
    for n in range(nsteps):
        g.fill_ghost(1, n * dt)
        cg = g.advance_level(1, dt)
        o.fill_ghost(1, n * dt)
        co = o.advance_level(1, dt)
        assert cg == co, (n, cg, co)
        if check_every and (n + 1) % check_every == 0:
            assert rel_err(g.read_level(1), o.read_level(1)) <= TOL, n
    return rel_err(g.read_level(1), o.read_level(1))


def dt_for(aux, descs, nu=0.8):
    return nu * min(float(descs["dx"][0]), float(descs["dy"][0])) / W.max_sound_speed(aux, descs)


@pytest.mark.parametrize("limiter", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("ot", [0, 1, 2])
@pytest.mark.parametrize("bc", [W.EXTRAP, W.PERIODIC])
def test_vc_random_media_every_limiter(limiter, ot, bc):
    """3 x 2 patches of 16 x 12 (ragged strips: 48 columns = 30 + 18), random
    media and data, 10 steps."""
    d = W.uniform_level(3, 2, 16, 12)
    seed = 10 * limiter + ot + (50 if bc == W.PERIODIC else 0)
    aux = W.random_media(d, seed)
    q0 = W.random_ic(d, seed)
    g, o = pair(d, q0, aux, limiter, ot, bc)
    err = run(g, o, 10, dt_for(aux, d))
    g.close()
    assert err <= TOL, err


def test_vc_layered_ring_100_steps():
    """The layered medium of the vc bench line (4 layers, impedance jumps up
    to 4x, an inclusion) on 4 x 4 patches of 64^2, ring pulse, MC, 100 steps
    at CFL 0.9 of the fastest layer."""
    d = W.uniform_level(4, 4, 64, 64)
    aux = W.media_field(d)
    g, o = pair(d, W.ring_ic(d), aux)
    err = run(g, o, 100, dt_for(aux, d, 0.9), check_every=25)
    g.close()
    assert err <= TOL, err


def test_vc_random_media_100_steps_periodic():
    d = W.uniform_level(2, 3, 32, 20)
    aux = W.random_media(d, 7, 0.3, 3.0)
    g, o = pair(d, W.random_ic(d, 7), aux, 4, 2, W.PERIODIC)
    err = run(g, o, 100, dt_for(aux, d, 0.9), check_every=50)
    g.close()
    assert err <= TOL, err


@pytest.mark.parametrize("th", ["64", "128"])
def test_vc_tiles_spanning_patch_rows(th):
    """Grid tiles of 64 / 128 rows over patches 16 rows tall (the bench's
    spanning-tile configuration), 20 steps."""
    d = W.uniform_level(4, 8, 24, 16)
    aux = W.media_field(d)
    os.environ["CLAW_GRID_TH"] = th
    try:
        g, o = pair(d, W.random_ic(d, 3), aux)
    finally:
        os.environ.pop("CLAW_GRID_TH")
    err = run(g, o, 20, dt_for(aux, d))
    g.close()
    assert err <= TOL, err


def test_vc_degenerate_shapes():
    """1-wide and 1-tall patches, a single 5 x 3 patch, 33-wide patches
    (strips of 30 + 3 columns)."""
    for npx, npy, mx, my in ((4, 2, 1, 32), (2, 4, 32, 1), (1, 1, 5, 3), (2, 2, 33, 32)):
        d = W.uniform_level(npx, npy, mx, my)
        aux = W.random_media(d, mx + my)
        g, o = pair(d, W.random_ic(d, mx * my), aux)
        err = run(g, o, 6, dt_for(aux, d))
        g.close()
        assert err <= TOL, (npx, npy, mx, my, err)


def test_vc_patch_cfl_matches_oracle():
    d = W.uniform_level(4, 3, 16, 8)
    aux = W.random_media(d, 11, 0.2, 4.0)
    g, o = pair(d, W.random_ic(d, 11), aux)
    run(g, o, 2, dt_for(aux, d))
    for p in range(len(d)):
        assert g.patch_cfl(1, p) == o.patch_cfl(1, p), p
    g.close()


def test_vc_constant_medium_matches_constant_kernel():
    """The vc kernel on a constant medium vs the constant-coefficient grid
    kernel (different arithmetic: same result to rounding)."""
    rho, K = 2.0, 0.5
    d = W.uniform_level(3, 3, 32, 32, rho=rho, K=K)
    n = int(d["mx"][0] * d["my"][0])
    aux = np.concatenate([np.concatenate([np.full(n, rho), np.full(n, K)]) for _ in d])
    q0 = W.random_ic(d, 5)
    dt = 0.9 * float(d["dx"][0]) / np.sqrt(K / rho)
    a = binding.Claw(W.DOMAIN, W.EXTRAP, 4, 2, device=0)
    a.set_level(1, d, q0)
    a.set_aux(1, aux)
    b = binding.Claw(W.DOMAIN, W.EXTRAP, 4, 2, device=0)
    b.set_level(1, d, q0)
    for k in range(30):
        a.fill_ghost(1, k * dt)
        b.fill_ghost(1, k * dt)
        assert a.advance_level(1, dt) == b.advance_level(1, dt)
    assert rel_err(a.read_level(1), b.read_level(1)) <= 1e-13
    a.close()
    b.close()


def sampled_vc_steps(patches_per_side, m, nsteps, samples_per_step, seed):
    """Full-size layered-medium level in the bench's launch configuration:
    before each of nsteps steps, sampled 3 x 3 patch blocks of the GPU state
    are read; the oracle's one step of each block (with the same medium)
    must equal the GPU's next state on the centre patch."""
    wl = W.c5_layered(patches_per_side, m)
    d = wl.levels[0].descs
    npx = patches_per_side
    g = binding.Claw(W.DOMAIN, W.EXTRAP, 4, 2, device=0)
    g.set_level(1, d, W.random_ic(d, seed))
    g.set_aux(1, W.media_field(d))
    dx = float(d["dx"][0])
    dt = 0.9 * dx / wl.extra["cmax"]
    rng = np.random.default_rng(seed)
    edge = [(0, 0), (npx - 1, npx - 1), (0, npx - 1), (npx - 1, 0)]
    checked = 0
    for n in range(nsteps):
        samples = [tuple(x) for x in rng.integers(0, npx, (samples_per_step, 2))] + [edge[n % len(edge)]]
        blocks = {}
        for pj, pi in samples:
            for b in range(max(pj - 1, 0), min(pj + 2, npx)):
                for a in range(max(pi - 1, 0), min(pi + 2, npx)):
                    blocks[(a, b)] = g.read(1, b * npx + a).copy()
        g.fill_ghost(1, n * dt)
        cfl = g.advance_level(1, dt)
        assert cfl == (dt / dx) * wl.extra["cmax"]
        for pj, pi in samples:
            js = range(max(pj - 1, 0), min(pj + 2, npx))
            iis = range(max(pi - 1, 0), min(pi + 2, npx))
            dom = (-1 + iis[0] * m * dx, -1 + (iis[-1] + 1) * m * dx,
                   -1 + js[0] * m * dx, -1 + (js[-1] + 1) * m * dx)
            boxes = [(a, b) for b in js for a in iis]
            sub = np.concatenate([W.make_descs([(a - iis[0]) * m], [(b - js[0]) * m], m, m, dx, dx, dom)
                                  for a, b in boxes])
            # the medium at the same cell centres (the full level's descriptors)
            full = np.concatenate([d[b * npx + a:b * npx + a + 1] for a, b in boxes])
            o = oracle.Oracle(dom, W.EXTRAP, 4, 2, nthreads=1)
            o.set_level(1, sub, np.concatenate([blocks[ab].ravel() for ab in boxes]))
            o.set_aux(1, W.media_field(full))
            o.fill_ghost(1, 0.0)
            o.advance_level(1, dt)
            ref = o.read(1, boxes.index((pi, pj)))
            assert rel_err(g.read(1, pj * npx + pi), ref) <= TOL, (n, pi, pj)
            checked += 1
    g.close()
    return checked


def test_vc_c5_layered_full_size_sampled():
    """The vc bench line's workload (16,384^2 cells, 64^2 patches, layered
    medium), 3 consecutive steps, 4 sampled blocks each."""
    assert sampled_vc_steps(256, 64, 3, 3, 91) == 12
