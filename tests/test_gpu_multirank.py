"""Multi-rank path on ONE GPU: N contexts (world = N, one per virtual rank) in
one process, remote ghost cells moved through host memory with the external
exchange mode (claw_halo_pack / claw_halo_unpack) instead of NCCL.  Everything
the NCCL path runs on each rank -- Morton partition, send/receive plans, the
pack kernel, frame-buffer ghosts read by the generic step kernel, per-rank
CFL -- runs here, and the N-rank result must be bitwise equal to the 1-rank
result (halo values are exact copies, the max is exact)."""
import numpy as np
import pytest

from paper_1808_02638_b200 import binding, workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def layout(name):
    if name == "c5small":
        return W.c5(patches_per_side=8, mx=32).levels[0].descs
    if name == "c4small":
        return W.c4(patches_per_side=16).levels[0].descs
    return W.ragged_level(6, 90, 70, 30)


@pytest.mark.parametrize("world,name,bc,path", [(2, "c5small", W.EXTRAP, 0), (3, "ragged", W.PERIODIC, 0),
                                                (4, "c4small", W.PERIODIC, 0), (8, "c5small", W.EXTRAP, 0),
                                                (5, "ragged", (1, 1, 2, 2), 0), (4, "c4small", W.PERIODIC, 1),
                                                (3, "c5small", (1, 1, 2, 2), 1)])
def test_virtual_ranks_bitwise_equal_single_rank(world, name, bc, path):
    d = layout(name)
    q0 = W.random_ic(d, world)
    offs = W.level_offsets(d)
    owners = binding.partition(d, world)
    ctxs = []
    for r in range(world):
        c = binding.Claw(W.DOMAIN, bc, 4, 2, device=0, rank=r, world=world, exchange=1, path=path)
        mine = np.concatenate([q0[offs[p]:offs[p + 1]] for p in range(len(d)) if owners[p] == r])
        c.set_level(1, d, mine)
        assert [c.owner(1, p) for p in range(len(d))] == list(owners)
        # uniform grids: band partition + table-free grid kernel on every rank
        assert c.level_mode(1) == ("generic" if name == "ragged" or path == 1 else "grid")
        ctxs.append(c)
    ref = binding.Claw(W.DOMAIN, bc, 4, 2, device=0)
    ref.set_level(1, d, q0)
    dx = float(min(d["dx"][0], d["dy"][0]))
    dt = 0.9 * dx
    moved = 0
    for n in range(6):
        for c in ctxs:
            c.fill_ghost(1, n * dt)
        for r in range(world):
            for s in range(world):
                if r != s:
                    buf = ctxs[r].halo_pack(1, s)
                    moved += buf.size
                    ctxs[s].halo_unpack(1, r, buf)
        cfl = max(c.advance_level(1, dt) for c in ctxs)
        ref.fill_ghost(1, n * dt)
        assert cfl == ref.advance_level(1, dt)
    assert moved > 0
    full = ref.read_level(1)
    got = np.empty_like(full)
    for r, c in enumerate(ctxs):
        mine = c.read_level(1)
        k = 0
        for p in range(len(d)):
            if owners[p] == r:
                n = offs[p + 1] - offs[p]
                got[offs[p]:offs[p + 1]] = mine[k:k + n]
                k += n
    assert np.array_equal(got, full)


@pytest.mark.parametrize("world,npx,mx,bc", [(2, 8, 32, W.EXTRAP), (3, 6, 16, W.PERIODIC), (4, 8, 32, (1, 1, 2, 2))])
def test_virtual_ranks_variable_media_bitwise_equal_single_rank(world, npx, mx, bc):
    """Variable media (claw_set_aux, R20) on a band-partitioned uniform grid:
    every rank gets the whole medium, keeps its band and the (Z, c) of its
    four halo rows; q halos move through the external exchange.  The N-rank
    run is bitwise the 1-rank run, CFLs included (a per-face max, exact)."""
    d = W.uniform_level(npx, npx, mx, mx)
    q0 = W.random_ic(d, 7 * world)
    aux = W.random_media(d, 5 * world, 0.4, 2.5)
    offs = W.level_offsets(d)
    owners = binding.partition(d, world)
    ctxs = []
    for r in range(world):
        c = binding.Claw(W.DOMAIN, bc, 4, 2, device=0, rank=r, world=world, exchange=1)
        mine = np.concatenate([q0[offs[p]:offs[p + 1]] for p in range(len(d)) if owners[p] == r])
        c.set_level(1, d, mine)
        assert c.level_mode(1) == "grid"
        c.set_aux(1, aux)
        ctxs.append(c)
    ref = binding.Claw(W.DOMAIN, bc, 4, 2, device=0)
    ref.set_level(1, d, q0)
    ref.set_aux(1, aux)
    dt = 0.8 * float(d["dx"][0]) / W.max_sound_speed(aux, d)
    for n in range(6):
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
        mine = c.read_level(1)
        want = np.concatenate([full[offs[p]:offs[p + 1]] for p in range(len(d)) if owners[p] == r])
        assert np.array_equal(mine, want)
        for p in range(len(d)):
            if owners[p] == r:
                assert c.patch_cfl(1, p) == ref.patch_cfl(1, p)


@pytest.mark.parametrize("world,npx,mx,tile_rows,bc,media", [
    (2, 16, 32, 0, W.EXTRAP, False), (4, 16, 32, 64, W.PERIODIC, False), (4, 16, 32, 96, (1, 1, 2, 2), False),
    (3, 12, 16, 48, W.EXTRAP, False), (2, 8, 64, 128, W.PERIODIC, False), (8, 16, 32, 32, W.EXTRAP, False),
    (4, 16, 32, 64, W.EXTRAP, True), (2, 8, 64, 128, (1, 1, 2, 2), True),
    # interior heights that are multiples of 4 but not of my: tiles start
    # anywhere in a patch row and the prologue / first prefetch cross patch rows
    (4, 16, 32, 20, W.EXTRAP, False), (2, 16, 32, 36, W.PERIODIC, False), (4, 16, 32, 60, (1, 1, 2, 2), False),
    (2, 8, 64, 124, W.EXTRAP, False), (4, 16, 32, 28, W.EXTRAP, True), (2, 8, 64, 100, W.PERIODIC, True)])
def test_band_split_tiles_bitwise_equal_single_rank(world, npx, mx, tile_rows, bc, media, monkeypatch):
    """Band split: each rank's step is an interior
    launch over rows [Y0 + 4, Y1 - 4) -- tiles of tile_rows rows that start 4
    rows into a patch row and span patch rows -- and an edge launch of the 4
    rows at each end of the band, after the halo.  With the grid kernel and
    the variable-media kernel, N ranks are bitwise the one-rank run.
    tile_rows: the interior tile height (CLAW_GRID_TH; 0 = the makespan rule)."""
    if tile_rows:
        monkeypatch.setenv("CLAW_GRID_TH", str(tile_rows))
    d = W.uniform_level(npx, npx, mx, mx)
    q0 = W.random_ic(d, 11 * world + mx)
    aux = W.random_media(d, 3 * world, 0.4, 2.5) if media else None
    offs = W.level_offsets(d)
    owners = binding.partition(d, world)
    ctxs = []
    for r in range(world):
        c = binding.Claw(W.DOMAIN, bc, 4, 2, device=0, rank=r, world=world, exchange=1)
        c.set_level(1, d, np.concatenate([q0[offs[p]:offs[p + 1]] for p in range(len(d)) if owners[p] == r]))
        assert c.level_mode(1) == "grid"
        if media:
            c.set_aux(1, aux)
        ctxs.append(c)
    ref = binding.Claw(W.DOMAIN, bc, 4, 2, device=0)
    ref.set_level(1, d, q0)
    dt = 0.9 * float(d["dx"][0])
    if media:
        ref.set_aux(1, aux)
        dt = 0.8 * float(d["dx"][0]) / W.max_sound_speed(aux, d)
    for n in range(5):
        for c in ctxs:
            c.fill_ghost(1, n * dt)
        for r in range(world):
            for s in range(world):
                if r != s:
                    ctxs[s].halo_unpack(1, r, ctxs[r].halo_pack(1, s))
        st0 = [c.stats()["step_launches"] for c in ctxs]
        cfl = max(c.advance_level(1, dt) for c in ctxs)
        # two launches per rank and step: interior tiles, then edge tiles
        assert [c.stats()["step_launches"] - s0 for c, s0 in zip(ctxs, st0)] == [2] * world
        ref.fill_ghost(1, n * dt)
        assert cfl == ref.advance_level(1, dt)
    full = ref.read_level(1)
    for r, c in enumerate(ctxs):
        want = np.concatenate([full[offs[p]:offs[p + 1]] for p in range(len(d)) if owners[p] == r])
        assert np.array_equal(c.read_level(1), want), r
    ref.close()
    for c in ctxs:
        c.close()
