"""GPU parity: libclaw.so (sm_100a) vs the CPU oracle, through the C-ABI.

Bar (BASELINE.json north_star): max|q_gpu - q_oracle| <= 1e-12 * max|q_oracle|
after 100 steps; CFL to 1e-14 relative (we require bitwise: the CFL is a max of
exact products).  Ghost frames (pure copies / same-order interpolation) must be
bitwise equal.  Arithmetic-invariance (tile shape, patch split) must be
bitwise.  Sizes span several tiles and ragged tails; the full C4 size is
checked on sampled patches the oracle can compute one by one.
"""
import math

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


def run_both(descs, q0, nsteps, dt, bc=W.EXTRAP, limiter=4, order_trans=2, domain=W.DOMAIN,
             tile_rows=0, check_cfl=True):
    g = binding.Claw(domain, bc, limiter, order_trans, device=0, tile_rows=tile_rows)
    g.set_level(1, descs, q0)
    o = oracle.Oracle(domain, bc, limiter, order_trans, nthreads=0)
    o.set_level(1, descs, q0)
    for n in range(nsteps):
        g.fill_ghost(1, n * dt)
        cg = g.advance_level(1, dt)
        o.fill_ghost(1, n * dt)
        co = o.advance_level(1, dt)
        if check_cfl:
            assert cg == co, (n, cg, co)
    qg, qo = g.read_level(1), o.read_level(1)
    g.close()
    return qg, qo


def rel_err(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def test_c1_ring_20_steps():
    wl = W.c1()
    d = wl.levels[0].descs
    qg, qo = run_both(d, W.ring_ic(d), 20, wl.dt0())
    assert rel_err(qg, qo) <= TOL


@pytest.mark.parametrize("limiter", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("order_trans", [0, 1, 2])
@pytest.mark.parametrize("bc", [W.EXTRAP, W.PERIODIC])
def test_ragged_level_random_data(limiter, order_trans, bc):
    d = W.ragged_level(11, 70, 45, 40)
    q0 = W.random_ic(d, limiter + 5 * order_trans)
    dx = float(d["dx"][0])
    dt = (0.9 if order_trans else 0.45) * dx
    qg, qo = run_both(d, q0, 20, dt, bc=bc, limiter=limiter, order_trans=order_trans)
    assert rel_err(qg, qo) <= TOL


@pytest.mark.parametrize("seed", range(5))
def test_ragged_level_mc_100_steps(seed):
    d = W.ragged_level(seed, 96, 80, 40)
    q0 = W.random_ic(d, seed)
    qg, qo = run_both(d, q0, 100, 0.9 * float(d["dx"][0]))
    assert rel_err(qg, qo) <= TOL


def test_c4_reduced_100_steps():
    wl = W.c4(patches_per_side=32)       # 1024 patches of 32^2, 1M cells
    d = wl.levels[0].descs
    qg, qo = run_both(d, W.ring_ic(d), 100, wl.dt0())
    assert rel_err(qg, qo) <= TOL


def test_c5_reduced_100_steps():
    wl = W.c5(patches_per_side=8)        # 512^2 cells as 64^2 patches
    d = wl.levels[0].descs
    qg, qo = run_both(d, W.random_ic(d, 3), 100, wl.dt0())
    assert rel_err(qg, qo) <= TOL


def test_tiny_and_degenerate_patches():
    # 1-wide and 1-tall patches, widths > 32 (two strips + ragged strip), 33x70
    boxes = [(0, 0, 1, 5), (1, 0, 33, 5), (34, 0, 6, 1), (34, 1, 6, 4), (0, 5, 40, 70)]
    d = np.concatenate([W.make_descs([a], [b], w, h, 2 / 40, 2 / 75) for a, b, w, h in boxes])
    q0 = W.random_ic(d, 9)
    qg, qo = run_both(d, q0, 10, 0.9 * 2 / 75)
    assert rel_err(qg, qo) <= TOL


def test_dt_zero_and_constant_state():
    d = W.ragged_level(1, 30, 30, 12)
    q0 = W.random_ic(d, 1)
    g = binding.Claw(W.DOMAIN, W.EXTRAP, 4, 2, device=0)
    g.set_level(1, d, q0)
    g.fill_ghost(1, 0.0)
    assert g.advance_level(1, 0.0) == 0.0
    assert np.array_equal(g.read_level(1), q0)
    const = np.concatenate([np.repeat([0.3, -1.2, 2.5], int(m * n)) for m, n in zip(d["mx"], d["my"])])
    g.write_level(1, const)
    g.fill_ghost(1, 0.0)
    g.advance_level(1, 0.05)
    assert np.array_equal(g.read_level(1), const)


@pytest.mark.parametrize("bc", [W.EXTRAP, W.PERIODIC, (1, 1, 2, 2)])
def test_ghost_frames_bitwise(bc):
    d = W.ragged_level(4, 50, 44, 20)
    q0 = W.random_ic(d, 4)
    g = binding.Claw(W.DOMAIN, bc, 4, 2, device=0)
    g.set_level(1, d, q0)
    g.fill_ghost(1, 0.0)
    o = oracle.Oracle(W.DOMAIN, bc, 4, 2)
    o.set_level(1, d, q0)
    o.fill_ghost(1, 0.0)
    for p in range(len(d)):
        assert np.array_equal(g.read_padded(1, p), o.read_padded(1, p)), p


@pytest.mark.parametrize("limiter", [1, 4])
def test_hand_examples_bitwise(limiter):
    q = np.zeros((3, 4, 4))
    q[0, :, :2] = 1.0
    dom = (0.0, 4.0, 0.0, 4.0)
    g = binding.Claw(dom, W.EXTRAP, limiter, 2, device=0)
    g.set_level(1, W.make_descs([0], [0], 4, 4, 1.0, 1.0, dom), q.ravel())
    g.fill_ghost(1, 0.0)
    assert g.advance_level(1, 0.5) == 0.5
    out = g.read(1, 0)
    assert np.array_equal(out[0], np.tile([1.0, 0.75, 0.25, 0.0], (4, 1)))
    assert np.array_equal(out[1], np.tile([0.0, 0.25, 0.25, 0.0], (4, 1)))
    q = np.zeros((3, 5, 5))
    q[0, 2, 2] = 1.0
    dom = (0.0, 5.0, 0.0, 5.0)
    g = binding.Claw(dom, W.EXTRAP, 4, 2, device=0)
    g.set_level(1, W.make_descs([0], [0], 5, 5, 1.0, 1.0, dom), q.ravel())
    g.fill_ghost(1, 0.0)
    g.advance_level(1, 0.5)
    out = g.read(1, 0)
    assert np.array_equal(out[0][1:4, 1:4], np.array([[1, 2, 1], [2, 4, 2], [1, 2, 1]]) / 16.0)
    assert out[0].sum() == 1.0


def test_tile_shape_and_patch_split_invariance_bitwise():
    n = 96
    big = W.uniform_level(1, 1, n, n)
    q0 = W.random_ic(big, 7)
    dt = 0.9 * 2 / n
    res = []
    for tr in (0, 16, 7):
        g = binding.Claw(W.DOMAIN, W.EXTRAP, 4, 2, device=0, tile_rows=tr)
        g.set_level(1, big, q0)
        for s in range(4):
            g.fill_ghost(1, s * dt)
            g.advance_level(1, dt)
        res.append(g.read_level(1))
        g.close()
    assert np.array_equal(res[0], res[1]) and np.array_equal(res[0], res[2])
    split = W.uniform_level(3, 4, 32, 24)
    full = q0.reshape(3, n, n)
    qs = np.concatenate([full[:, b:b + 24, a:a + 32].ravel()
                         for b in range(0, n, 24) for a in range(0, n, 32)])
    g = binding.Claw(W.DOMAIN, W.EXTRAP, 4, 2, device=0)
    g.set_level(1, split, qs)
    for s in range(4):
        g.fill_ghost(1, s * dt)
        g.advance_level(1, dt)
    got = g.read_level(1)
    ref = res[0].reshape(3, n, n)
    k = 0
    for b in range(0, n, 24):
        for a in range(0, n, 32):
            blk = got[k:k + 3 * 24 * 32].reshape(3, 24, 32)
            assert np.array_equal(blk, ref[:, b:b + 24, a:a + 32])
            k += 3 * 24 * 32


def test_conservation_and_symmetry_at_full_c4_size():
    """Properties that hold at any size (full C4, 65,536 patches of 32^2):
    radial symmetry of the ring and cfl = c dt / dx."""
    wl = W.c4()
    d = wl.levels[0].descs
    g = binding.Claw(W.DOMAIN, W.EXTRAP, 4, 2, device=0)
    g.set_level(1, d, W.ring_ic(d))
    dt = wl.dt0()
    for s in range(5):
        g.fill_ghost(1, s * dt)
        cfl = g.advance_level(1, dt)
    assert cfl == (dt / float(d["dx"][0])) * 1.0
    q = g.read_level(1).reshape(256, 256, 3, 32, 32)
    p = q[:, :, 0].transpose(0, 2, 1, 3).reshape(8192, 8192)
    u = q[:, :, 1].transpose(0, 2, 1, 3).reshape(8192, 8192)
    v = q[:, :, 2].transpose(0, 2, 1, 3).reshape(8192, 8192)
    tol = 8e-16 * np.abs(p).max() * 10
    assert np.abs(p - p.T).max() <= tol
    assert np.abs(u - v.T).max() <= tol
    assert np.abs(p - p[:, ::-1]).max() <= tol


def test_sampled_patches_at_full_c4_size_one_step():
    """Full C4 in the bench's launch configuration: after 3 GPU steps, one more
    step of sampled patches is recomputed by the oracle from the GPU's own
    state on the 3x3 block of patches around each sample."""
    wl = W.c4()
    d = wl.levels[0].descs
    g = binding.Claw(W.DOMAIN, W.EXTRAP, 4, 2, device=0)
    q0 = W.random_ic(d, 21)
    g.set_level(1, d, q0)
    dt = wl.dt0()
    for s in range(3):
        g.fill_ghost(1, s * dt)
        g.advance_level(1, dt)
    qn = g.read_level(1).reshape(len(d), 3, 32, 32)
    g.fill_ghost(1, 3 * dt)
    g.advance_level(1, dt)
    q1 = g.read_level(1).reshape(len(d), 3, 32, 32)
    rng = np.random.default_rng(0)
    samples = list(rng.integers(0, 256, (12, 2))) + [(0, 0), (255, 255), (0, 255), (128, 0)]
    dx = float(d["dx"][0])
    for pj, pi in samples:
        js = range(max(pj - 1, 0), min(pj + 2, 256))
        iis = range(max(pi - 1, 0), min(pi + 2, 256))
        dom = (-1 + iis[0] * 32 * dx, -1 + (iis[-1] + 1) * 32 * dx,
               -1 + js[0] * 32 * dx, -1 + (js[-1] + 1) * 32 * dx)
        boxes = [(a, b) for b in js for a in iis]
        sub = np.concatenate([W.make_descs([(a - iis[0]) * 32], [(b - js[0]) * 32], 32, 32, dx, dx, dom)
                              for a, b in boxes])
        qsub = np.concatenate([qn[b * 256 + a].ravel() for a, b in boxes])
        o = oracle.Oracle(dom, W.EXTRAP, 4, 2, nthreads=1)
        o.set_level(1, sub, qsub)
        o.fill_ghost(1, 0.0)
        o.advance_level(1, dt)
        k = boxes.index((pi, pj))
        ref = o.read(1, k)
        assert rel_err(q1[pj * 256 + pi], ref) <= TOL, (pi, pj)


def test_sampled_patches_at_full_c5_size_one_step():
    """The default bench workload at full size (C5: 16384^2 cells, 65,536
    patches of 64^2, 14.5 GB of state) in the bench's launch configuration
    (grid kernel, 256-row tiles spanning patch rows): after 3 GPU steps, one
    more step of sampled patches (corners, edges, random interior) is
    recomputed by the oracle from the GPU's own state on the 3x3 block of
    patches around each sample; patches are read one by one."""
    wl = W.c5()
    d = wl.levels[0].descs
    g = binding.Claw(W.DOMAIN, W.EXTRAP, 4, 2, device=0)
    g.set_level(1, d, W.random_ic(d, 55))
    assert g.level_mode(1) == "grid"
    dt = wl.dt0()
    for s in range(3):
        g.fill_ghost(1, s * dt)
        g.advance_level(1, dt)
    rng = np.random.default_rng(5)
    samples = [tuple(x) for x in rng.integers(0, 256, (10, 2))] + [(0, 0), (255, 255), (0, 255), (255, 0), (3, 128)]
    blocks = {}
    for pj, pi in samples:
        for b in range(max(pj - 1, 0), min(pj + 2, 256)):
            for a in range(max(pi - 1, 0), min(pi + 2, 256)):
                blocks[(a, b)] = g.read(1, b * 256 + a).copy()
    g.fill_ghost(1, 3 * dt)
    cfl = g.advance_level(1, dt)
    assert cfl == (dt / float(d["dx"][0])) * 1.0
    dx = float(d["dx"][0])
    for pj, pi in samples:
        js = range(max(pj - 1, 0), min(pj + 2, 256))
        iis = range(max(pi - 1, 0), min(pi + 2, 256))
        dom = (-1 + iis[0] * 64 * dx, -1 + (iis[-1] + 1) * 64 * dx,
               -1 + js[0] * 64 * dx, -1 + (js[-1] + 1) * 64 * dx)
        boxes = [(a, b) for b in js for a in iis]
        sub = np.concatenate([W.make_descs([(a - iis[0]) * 64], [(b - js[0]) * 64], 64, 64, dx, dx, dom)
                              for a, b in boxes])
        o = oracle.Oracle(dom, W.EXTRAP, 4, 2, nthreads=1)
        o.set_level(1, sub, np.concatenate([blocks[ab].ravel() for ab in boxes]))
        o.fill_ghost(1, 0.0)
        o.advance_level(1, dt)
        ref = o.read(1, boxes.index((pi, pj)))
        assert rel_err(g.read(1, pj * 256 + pi), ref) <= TOL, (pi, pj)
    g.close()


def run_hierarchy(wl, n_coarse, q0s, use_gpu, update=False):
    ratios = {L + 1: wl.levels[L + 1].ratio for L in range(len(wl.levels) - 1)}
    nlev = len(wl.levels)
    if use_gpu:
        h = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0)
    else:
        h = oracle.Oracle(wl.domain, wl.bc, wl.limiter, wl.order_trans, nthreads=0)
    for L, (lv, q0) in enumerate(zip(wl.levels, q0s), start=1):
        h.set_level(L, lv.descs, q0)

    def bo(level, t, dt):
        h.fill_ghost(level, t)
        c = h.advance_level(level, dt)
        if level < nlev:
            R = ratios[level]
            for k in range(R):
                c = max(c, bo(level + 1, t + k * dt / R, dt / R))
            if update:          # fine level caught up -> average onto coarse
                h.update_level(level + 1)
        return c

    dt = wl.dt0()
    cfls = [bo(1, n * dt, dt) for n in range(n_coarse)]
    out = [h.read_level(L) for L in range(1, nlev + 1)]
    return out, cfls


@pytest.mark.parametrize("name,steps", [("c2", 10), ("c3", 2)])
def test_multilevel_berger_oliger(name, steps):
    wl = getattr(W, name)()
    q0s = W.hierarchy_ic(wl)
    qg, cg = run_hierarchy(wl, steps, q0s, True)
    qo, co = run_hierarchy(wl, steps, q0s, False)
    assert cg == co
    for a, b in zip(qg, qo):
        assert rel_err(a, b) <= TOL


def test_coarse_interp_ghost_frames_bitwise():
    wl = W.c2()
    q0s = [W.random_ic(L.descs, 5 + k) for k, L in enumerate(wl.levels)]
    g = binding.Claw(wl.domain, wl.bc, 4, 2, device=0)
    o = oracle.Oracle(wl.domain, wl.bc, 4, 2)
    for L, (lv, q0) in enumerate(zip(wl.levels, q0s), start=1):
        g.set_level(L, lv.descs, q0)
        o.set_level(L, lv.descs, q0)
    dt = wl.dt0()
    for h in (g, o):
        h.fill_ghost(1, 0.0)
        h.advance_level(1, dt)
    # both time levels of level 1 must hold identical bytes: give the GPU the
    # oracle's q^{n+1} (the two steps differ by rounding, which is not what
    # this test is about)
    g.write_level(1, o.read_level(1))
    for t in (0.0, 0.25 * dt, 0.75 * dt):
        g.fill_ghost(2, t)
        o.fill_ghost(2, t)
        for p in range(len(wl.levels[1].descs)):
            assert np.array_equal(g.read_padded(2, p), o.read_padded(2, p)), (t, p)
    with pytest.raises(binding.ClawError) as e:
        g.fill_ghost(2, 2 * dt)
    assert e.value.code == binding.CLAW_ESTATE


def test_torch_stream_adoption():
    import torch
    s = torch.cuda.Stream()
    d = W.uniform_level(4, 4, 32, 32)
    q0 = W.ring_ic(d)
    g = binding.Claw(W.DOMAIN, W.EXTRAP, 4, 2, device=0, stream=s.cuda_stream)
    g.set_level(1, d, q0)
    g.set_profiling(True)
    for n in range(3):
        g.fill_ghost(1, 0.0)
        g.advance_level(1, 0.01)
    st = g.stats()
    assert st["step_launches"] == 3 and st["step_ms"] > 0 and st["cells_advanced"] == 3 * 16 * 1024


@pytest.mark.parametrize("npx,npy,mx,my,bc,limiter,ot", [
    (8, 8, 32, 32, W.EXTRAP, 4, 2), (4, 4, 64, 64, W.PERIODIC, 4, 2), (3, 5, 7, 5, W.EXTRAP, 1, 2),
    (5, 3, 13, 70, (2, 2, 1, 1), 2, 1), (2, 2, 33, 31, (1, 1, 2, 2), 0, 0), (1, 1, 61, 3, W.EXTRAP, 3, 2)])
def test_grid_kernel_bitwise_equals_generic_kernel(npx, npy, mx, my, bc, limiter, ot):
    """The table-free grid kernel (uniform levels) and the generic ghost-table
    kernel run the same cell arithmetic: results must agree bit for bit, and
    both must match the oracle."""
    d = W.uniform_level(npx, npy, mx, my)
    q0 = W.random_ic(d, npx * 100 + mx)
    dt = (0.9 if ot else 0.45) * 2 / max(npx * mx, npy * my)
    res = []
    for path in (0, 1):
        g = binding.Claw(W.DOMAIN, bc, limiter, ot, device=0, path=path)
        g.set_level(1, d, q0)
        for n in range(6):
            g.fill_ghost(1, n * dt)
            c = g.advance_level(1, dt)
        res.append((g.read_level(1), c, g.patch_cfl(1, len(d) - 1)))
        g.close()
    assert np.array_equal(res[0][0], res[1][0])
    assert res[0][1] == res[1][1] and res[0][2] == res[1][2]
    qg, qo = run_both(d, q0, 6, dt, bc=bc, limiter=limiter, order_trans=ot)
    assert rel_err(qg, qo) <= TOL


def test_native_hierarchy_driver_equals_python_driver():
    """claw_advance_hierarchy (native subcycling, one host sync) runs the same
    level steps as the Python Berger-Oliger recursion: bitwise equal."""
    wl = W.c2()
    q0s = [W.random_ic(L.descs, 40 + k) for k, L in enumerate(wl.levels)]
    out = []
    for native in (True, False):
        g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0)
        for L, (lv, q0) in enumerate(zip(wl.levels, q0s), start=1):
            g.set_level(L, lv.descs, q0)
        dt = wl.dt0()
        cfl = []
        for n in range(3):
            if native:
                cfl.append(g.advance_hierarchy(n * dt, dt))
            else:
                cfl.append(binding.berger_oliger(g, 1, n * dt, dt, {1: 4}, 2))
        out.append((g.read_level(1), g.read_level(2), cfl))
        g.close()
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
    assert out[0][2] == out[1][2]


@pytest.mark.parametrize("name,steps", [("c2", 6), ("c3", 2)])
def test_multilevel_with_updating(name, steps):
    """Berger-Oliger with updating (NEXT-1): Python recursion on the GPU and
    the native claw_advance_hierarchy(update) both match the oracle."""
    wl = getattr(W, name)()
    q0s = W.hierarchy_ic(wl)
    qg, cg = run_hierarchy(wl, steps, q0s, True, update=True)
    qo, co = run_hierarchy(wl, steps, q0s, False, update=True)
    assert cg == co
    for a, b in zip(qg, qo):
        assert rel_err(a, b) <= TOL
    g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0)
    for L, (lv, q0) in enumerate(zip(wl.levels, q0s), start=1):
        g.set_level(L, lv.descs, q0)
    dt = wl.dt0()
    cn = [g.advance_hierarchy(n * dt, dt, update=True) for n in range(steps)]
    assert cn == cg
    for L in range(1, len(wl.levels) + 1):
        assert np.array_equal(g.read_level(L), qg[L - 1])


def test_update_level_bitwise_and_state_checks():
    wl = W.c2()
    q0s = [W.random_ic(L.descs, 70 + k) for k, L in enumerate(wl.levels)]
    g = binding.Claw(wl.domain, wl.bc, 4, 2, device=0)
    o = oracle.Oracle(wl.domain, wl.bc, 4, 2)
    for L, (lv, q0) in enumerate(zip(wl.levels, q0s), start=1):
        g.set_level(L, lv.descs, q0)
        o.set_level(L, lv.descs, q0)
    g.update_level(2)
    o.update_level(2)
    assert np.array_equal(g.read_level(1), o.read_level(1))
    g.fill_ghost(1, 0.0)
    g.advance_level(1, wl.dt0())
    with pytest.raises(binding.ClawError) as e:
        g.update_level(2)             # level 2 has not caught up
    assert e.value.code == binding.CLAW_ESTATE


def test_update_level_unaligned_fine_patches_bitwise():
    """Fine patches whose edges split coarse cells: the coarse cells whose
    children straddle two fine patches take the general (slow) path."""
    dom = (0.0, 1.0, 0.0, 1.0)
    cd = W.uniform_level(1, 1, 8, 8, dom)
    boxes = [(3, 3, 5, 4), (8, 3, 4, 4), (3, 7, 9, 3)]
    fd = np.concatenate([W.make_descs([a], [b], w, h, 1 / 16, 1 / 16, dom) for a, b, w, h in boxes])
    qc, qf = W.random_ic(cd, 1), W.random_ic(fd, 2)
    g = binding.Claw(dom, W.EXTRAP, 4, 2, device=0)
    o = oracle.Oracle(dom, W.EXTRAP, 4, 2)
    for h in (g, o):
        h.set_level(1, cd, qc)
        h.set_level(2, fd, qf)
        h.update_level(2)
    out = g.read_level(1)
    assert np.array_equal(out, o.read_level(1))
    assert not np.array_equal(out, qc)


@pytest.mark.parametrize("npx,npy,mx,my,th,bc", [
    (8, 8, 32, 32, 64, W.EXTRAP), (6, 5, 16, 16, 48, W.PERIODIC), (4, 7, 24, 8, 32, (2, 2, 1, 1)),
    (3, 3, 32, 32, 96, W.EXTRAP)])
def test_grid_tiles_spanning_patch_rows(npx, npy, mx, my, th, bc, monkeypatch):
    """Grid tiles of th > my rows (several patch rows; the kernel steps its row
    pointers across patch-row boundaries, ragged last tile): bitwise equal to
    the generic kernel."""
    d = W.uniform_level(npx, npy, mx, my)
    q0 = W.random_ic(d, 7 * mx + th)
    dt = 0.9 * 2 / max(npx * mx, npy * my)
    res = []
    for path in (0, 1):
        monkeypatch.setenv("CLAW_GRID_TH", str(th))
        g = binding.Claw(W.DOMAIN, bc, 4, 2, device=0, path=path)
        g.set_level(1, d, q0)
        assert g.level_mode(1) == ("grid" if path == 0 else "generic")
        for n in range(5):
            g.fill_ghost(1, n * dt)
            c = g.advance_level(1, dt)
        res.append((g.read_level(1), c))
        g.close()
    assert np.array_equal(res[0][0], res[1][0]) and res[0][1] == res[1][1]


@pytest.mark.parametrize("case", ["c3", "r2_periodic", "r4_extrap"])
def test_sparse_lattice_grid_kernel_bitwise_equals_generic(case):
    """A finer level of equal, lattice-aligned patches (not covering the
    domain) runs the grid kernel on a sparse lattice, its coarse ghost values
    in the lattice's empty slots: bitwise equal to the generic kernel, through
    hierarchy steps with updating."""
    if case == "c3":
        wl = W.c3()
        levels = [lv.descs for lv in wl.levels]
        q0s = W.hierarchy_ic(wl)
        dom, bc, nsteps = wl.domain, wl.bc, 2
    else:
        dom, nsteps = W.DOMAIN, 4
        if case == "r2_periodic":
            n1, R, mx, bc = 32, 2, 8, W.PERIODIC
            slots = [(x, y) for x in range(8) for y in range(8) if 2 <= x + y <= 11 and (3 * x + y) % 4 != 0]
        else:
            n1, R, mx, bc = 16, 4, 16, W.EXTRAP
            slots = [(0, 0), (1, 0), (1, 1), (2, 1), (3, 2), (3, 3)]
        d1 = W.uniform_level(2, 2, n1 // 2, n1 // 2, dom)
        dxf = (dom[1] - dom[0]) / n1 / R
        d2 = np.concatenate([W.make_descs([x * mx], [y * mx], mx, mx, dxf, dxf, dom) for x, y in slots])
        levels = [d1, d2]
        q0s = [W.random_ic(d1, 3), W.random_ic(d2, 4)]
    res = []
    for path in (0, 1):
        g = binding.Claw(dom, bc, 4, 2, device=0, path=path)
        for L, (d, q) in enumerate(zip(levels, q0s), start=1):
            g.set_level(L, d, q)
        assert g.level_mode(len(levels)) == ("sparse" if path == 0 else "generic")
        dt = 0.9 * float(levels[0]["dx"][0])
        cfl = [g.advance_hierarchy(n * dt, dt, update=True) for n in range(nsteps)]
        res.append(([g.read_level(L) for L in range(1, len(levels) + 1)], cfl))
        g.close()
    assert res[0][1] == res[1][1]
    for x, y in zip(res[0][0], res[1][0]):
        assert np.array_equal(x, y)
