"""The wide grid kernel (two columns per lane, 62-column strips; DESIGN.md §8
"step_grid2_kernel") against the 32-lane grid kernel (CLAW_GRID_WIDE=0) and the
generic ghost-table kernel: the three run the same cell arithmetic, so results
must agree bit for bit, and the wide one must match the oracle to the
north_star bar.  Shapes cover level widths below, at and around multiples of
the 62-column strip (ragged last strips, a one-strip level, the first strip's
virtual column -1), both BCs per axis, every limiter and order_trans, tiles
spanning patch rows, the sparse lattice and band-mode virtual ranks."""
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


def run(d, q0, bc, limiter, ot, nsteps, dt, path, wide, monkeypatch, th=None):
    monkeypatch.setenv("CLAW_GRID_WIDE", "1" if wide else "0")
    if th:
        monkeypatch.setenv("CLAW_GRID_TH", str(th))
    g = binding.Claw(W.DOMAIN, bc, limiter, ot, device=0, path=path)
    g.set_level(1, d, q0)
    mode = g.level_mode(1)
    cfl = []
    for n in range(nsteps):
        g.fill_ghost(1, n * dt)
        cfl.append(g.advance_level(1, dt))
    out = g.read_level(1)
    g.close()
    return out, cfl, mode


CASES = [
    # npx, npy, mx, my, bc, limiter, ot
    # (grid mode needs gapless patches: mx * my a multiple of 32)
    (1, 1, 2, 16, W.EXTRAP, 4, 2),           # NX = 2: one strip, almost all lanes clamped
    (1, 3, 60, 8, W.PERIODIC, 4, 2),         # NX = 60 < 62
    (1, 2, 62, 16, W.EXTRAP, 4, 2),          # NX = 62: the output needs two strips (column -1 offset)
    (2, 2, 32, 32, (2, 2, 1, 1), 4, 2),      # NX = 64
    (5, 4, 26, 16, W.PERIODIC, 1, 2),        # NX = 130 (ragged third strip)
    (4, 3, 32, 20, (1, 1, 2, 2), 2, 1),      # NX = 128
    (3, 3, 42, 16, W.EXTRAP, 3, 2),          # NX = 126
    (2, 5, 62, 16, W.PERIODIC, 0, 0),        # NX = 124 (exact two strips + 1 column)
    (8, 8, 32, 32, W.EXTRAP, 4, 2),          # specialised 32x32
    (4, 4, 64, 64, W.PERIODIC, 4, 2),        # specialised 64x64
    (3, 2, 64, 64, W.EXTRAP, 4, 1),          # 64x64 but order_trans 1: generic template
]


@pytest.mark.parametrize("npx,npy,mx,my,bc,limiter,ot", CASES)
def test_wide_equals_narrow_and_generic_bitwise(npx, npy, mx, my, bc, limiter, ot, monkeypatch):
    d = W.uniform_level(npx, npy, mx, my)
    q0 = W.random_ic(d, 31 * mx + my)
    dt = (0.9 if ot else 0.45) * 2 / max(npx * mx, npy * my)
    wide, cw, mw = run(d, q0, bc, limiter, ot, 5, dt, 0, True, monkeypatch)
    narrow, cn, mn = run(d, q0, bc, limiter, ot, 5, dt, 0, False, monkeypatch)
    gen, cg, mg = run(d, q0, bc, limiter, ot, 5, dt, 1, True, monkeypatch)
    assert (mw, mn, mg) == ("grid", "grid", "generic")
    assert np.array_equal(wide, narrow) and np.array_equal(wide, gen)
    assert cw == cn == cg
    o = oracle.Oracle(W.DOMAIN, bc, limiter, ot, nthreads=0)
    o.set_level(1, d, q0)
    for n in range(5):
        o.fill_ghost(1, n * dt)
        assert o.advance_level(1, dt) == cw[n]
    qo = o.read_level(1)
    assert float(np.abs(wide - qo).max() / np.abs(qo).max()) <= TOL


@pytest.mark.parametrize("npx,npy,mx,my,th,bc", [
    (8, 8, 32, 32, 64, W.EXTRAP), (6, 5, 16, 16, 48, W.PERIODIC), (4, 7, 24, 8, 32, (2, 2, 1, 1)),
    (3, 3, 32, 32, 96, W.EXTRAP), (5, 6, 32, 32, 256, W.PERIODIC)])
def test_wide_tiles_spanning_patch_rows(npx, npy, mx, my, th, bc, monkeypatch):
    d = W.uniform_level(npx, npy, mx, my)
    q0 = W.random_ic(d, 5 * mx + th)
    dt = 0.9 * 2 / max(npx * mx, npy * my)
    wide, cw, _ = run(d, q0, bc, 4, 2, 4, dt, 0, True, monkeypatch, th=th)
    narrow, cn, _ = run(d, q0, bc, 4, 2, 4, dt, 0, False, monkeypatch, th=th)
    assert np.array_equal(wide, narrow) and cw == cn


def test_wide_c5_reduced_100_steps_vs_oracle(monkeypatch):
    """The bench's kernel configuration (64x64 patches, MC, order_trans 2,
    256-row tiles spanning patch rows) on a 512^2 cut of C5 for 100 steps."""
    monkeypatch.setenv("CLAW_GRID_WIDE", "1")
    wl = W.c5(patches_per_side=8)
    d = wl.levels[0].descs
    q0 = W.ring_ic(d)
    dt = wl.dt0()
    g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0)
    g.set_level(1, d, q0)
    assert g.level_mode(1) == "grid"
    o = oracle.Oracle(wl.domain, wl.bc, wl.limiter, wl.order_trans, nthreads=0)
    o.set_level(1, d, q0)
    for n in range(100):
        g.fill_ghost(1, n * dt)
        o.fill_ghost(1, n * dt)
        assert g.advance_level(1, dt) == o.advance_level(1, dt)
    qg, qo = g.read_level(1), o.read_level(1)
    g.close()
    assert float(np.abs(qg - qo).max() / np.abs(qo).max()) <= TOL


def test_wide_sparse_lattice_c3(monkeypatch):
    """C3's level 3 (1,676 patches of 32^2 on a 50x50 lattice) on the wide
    kernel: bitwise equal to the narrow grid kernel through hierarchy steps."""
    wl = W.c3()
    levels = [lv.descs for lv in wl.levels]
    q0s = W.hierarchy_ic(wl)
    res = []
    for wide in (True, False):
        monkeypatch.setenv("CLAW_GRID_WIDE", "1" if wide else "0")
        g = binding.Claw(wl.domain, wl.bc, 4, 2, device=0)
        for L, (d, q) in enumerate(zip(levels, q0s), start=1):
            g.set_level(L, d, q)
        assert g.level_mode(3) == "sparse"
        dt = 0.9 * float(levels[0]["dx"][0])
        cfl = [g.advance_hierarchy(n * dt, dt, update=True) for n in range(2)]
        res.append(([g.read_level(L) for L in range(1, 4)], cfl))
        g.close()
    assert res[0][1] == res[1][1]
    for x, y in zip(res[0][0], res[1][0]):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("world,bc", [(2, W.EXTRAP), (3, W.PERIODIC), (4, (1, 1, 2, 2))])
def test_wide_band_mode_virtual_ranks(world, bc, monkeypatch):
    """Band mode (multi-rank uniform level): each virtual rank runs the wide
    kernel on its band with halo rows from the frame; bitwise equal to one
    rank."""
    monkeypatch.setenv("CLAW_GRID_WIDE", "1")
    d = W.c5(patches_per_side=6, mx=32).levels[0].descs
    q0 = W.random_ic(d, 40 + world)
    offs = W.level_offsets(d)
    owners = binding.partition(d, world)
    ctxs = []
    for r in range(world):
        c = binding.Claw(W.DOMAIN, bc, 4, 2, device=0, rank=r, world=world, exchange=1)
        c.set_level(1, d, np.concatenate([q0[offs[p]:offs[p + 1]] for p in range(len(d)) if owners[p] == r]))
        assert c.level_mode(1) == "grid"
        ctxs.append(c)
    ref = binding.Claw(W.DOMAIN, bc, 4, 2, device=0)
    ref.set_level(1, d, q0)
    dt = 0.9 * float(d["dx"][0])
    for n in range(4):
        for c in ctxs:
            c.fill_ghost(1, n * dt)
        for r in range(world):
            for s in range(world):
                if r != s:
                    ctxs[s].halo_unpack(1, r, ctxs[r].halo_pack(1, s))
        cfl = max(c.advance_level(1, dt) for c in ctxs)
        ref.fill_ghost(1, n * dt)
        assert cfl == ref.advance_level(1, dt)
    full = ref.read_level(1)
    for r, c in enumerate(ctxs):
        mine = np.concatenate([full[offs[p]:offs[p + 1]] for p in range(len(d)) if owners[p] == r])
        assert np.array_equal(c.read_level(1), mine)
    for c in ctxs + [ref]:
        c.close()
