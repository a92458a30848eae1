"""The library's NCCL code path with several PROCESSES on one GPU.

Real NCCL refuses two ranks on one GPU ("Duplicate GPU detected",
profiles/r01_nccl_dup_probe.txt), so libclaw is pointed (CLAW_NCCL_LIB) at a
test stand-in (tests/nccl_shim/ncclshim.c) that implements the calls libclaw
makes -- unique id, communicator init/destroy, grouped send/recv, float64 max
all-reduce -- between processes through a memory-mapped file with synchronous
device<->host copies.  Everything else is the production multi-rank path:
claw_create with world > 1 and the NCCL exchange, the partition, the pack
kernel on the comm stream, receives straight into the frame, the event that
gates the edge tiles after the interior tiles, and the CFL all-reduce inside
claw_advance_level.  Each rank's owned patches after several steps must be
bitwise equal to a one-rank run, and every rank must return the global CFL."""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1808_02638_b200 import binding, workloads as W

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM_SRC = os.path.join(ROOT, "tests", "nccl_shim", "ncclshim.c")

WORKER = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1808_02638_b200 import binding, workloads as W
rank, world, idhex, name, bcs, out = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5], sys.argv[6], sys.argv[7]
driver = sys.argv[8]
bc = tuple(int(x) for x in bcs.split(","))
d = W.c5(patches_per_side=6, mx=32).levels[0].descs if name in ("uniform", "vc") else W.ragged_level(6, 90, 70, 30)
q0 = W.random_ic(d, 77)
offs = W.level_offsets(d)
owners = binding.partition(d, world)
g = binding.Claw(W.DOMAIN, bc, 4, 2, device=0, rank=rank, world=world, nccl_id=bytes.fromhex(idhex))
g.set_level(1, d, np.concatenate([q0[offs[p]:offs[p + 1]] for p in range(len(d)) if owners[p] == rank]))
dt = 0.9 * float(d["dx"][0])
if name == "vc":
    aux = W.media_field(d)
    g.set_aux(1, aux)
    dt /= W.max_sound_speed(aux, d)
cfl = []
if driver == "batch":
    cfl = g.advance_hierarchy_n(0.0, dt, 5).tolist()
else:
    for n in range(5):
        g.fill_ghost(1, n * dt)
        cfl.append(g.advance_level(1, dt))
np.save(out, g.read_level(1))
np.save(out + ".cfl.npy", np.array(cfl))
print("mode", g.level_mode(1))
g.close()
'''


@pytest.fixture(scope="module")
def shim(tmp_path_factory):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = str(tmp_path_factory.mktemp("shim") / "libncclshim.so")
    subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-o", out, SHIM_SRC, "-ldl"], check=True)
    return out


@pytest.mark.parametrize("world,name,bc,driver", [(2, "uniform", W.EXTRAP, "level"), (3, "uniform", W.PERIODIC, "level"),
                                                  (2, "ragged", W.PERIODIC, "level"),
                                                  (4, "ragged", (1, 1, 2, 2), "level"),
                                                  (3, "uniform", W.EXTRAP, "batch"),
                                                  (2, "ragged", W.PERIODIC, "batch"),
                                                  (4, "vc", W.EXTRAP, "level"), (4, "vc", W.EXTRAP, "batch")])
def test_nccl_path_processes_bitwise_equal_single_rank(shim, tmp_path, world, name, bc, driver):
    """driver "level": claw_advance_level per step (the CFL all-reduce of
    every level step); "batch": claw_advance_hierarchy_n of the single level
    (K steps per host synchronisation, one all-reduce of the K per-step CFLs
    at the end).  "vc": a layered medium whose max sound speed differs
    between the ranks' bands, so only the reduction gives every rank the
    global CFL."""
    env = dict(os.environ, CLAW_NCCL_LIB=shim)
    # the unique id comes from the same library call rank 0 would make
    gen = subprocess.run([sys.executable, "-c",
                          "import sys; sys.path.insert(0, sys.argv[1]); "
                          "from paper_1808_02638_b200 import binding; print(binding.nccl_unique_id().hex())", ROOT],
                         env=env, capture_output=True, text=True, check=True)
    idhex = gen.stdout.strip().splitlines()[-1]
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    bcs = ",".join(str(x) for x in bc)
    procs = [subprocess.Popen([sys.executable, str(script), ROOT, str(r), str(world), idhex, name, bcs,
                               str(tmp_path / f"rank{r}.npy"), driver], env=env, stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for r in range(world)]
    outs = [p.communicate(timeout=600) for p in procs]
    for p, (so, se) in zip(procs, outs):
        assert p.returncode == 0, se[-3000:]
    modes = {so.strip().splitlines()[-1] for so, _ in outs}
    assert modes == {"mode generic" if name == "ragged" else "mode grid"}, modes
    # the one-rank reference
    d = W.c5(patches_per_side=6, mx=32).levels[0].descs if name in ("uniform", "vc") else W.ragged_level(6, 90, 70, 30)
    q0 = W.random_ic(d, 77)
    offs = W.level_offsets(d)
    owners = binding.partition(d, world)
    ref = binding.Claw(W.DOMAIN, bc, 4, 2, device=0)
    ref.set_level(1, d, q0)
    dt = 0.9 * float(d["dx"][0])
    if name == "vc":
        aux = W.media_field(d)
        ref.set_aux(1, aux)
        dt /= W.max_sound_speed(aux, d)
    cfl = []
    for n in range(5):
        ref.fill_ghost(1, n * dt)
        cfl.append(ref.advance_level(1, dt))
    full = ref.read_level(1)
    ref.close()
    for r in range(world):
        mine = np.concatenate([full[offs[p]:offs[p + 1]] for p in range(len(d)) if owners[p] == r])
        assert np.array_equal(np.load(tmp_path / f"rank{r}.npy"), mine), r
        assert np.load(tmp_path / f"rank{r}.npy.cfl.npy").tolist() == cfl
    if name == "vc":  # the bands' own maxima differ: the CFL really was reduced
        local = []
        for r in range(world):
            sub = d[owners == r]
            ao = offs // 3 * 2   # (rho, K) per cell; offs counts (p, u, v)
            a_r = np.concatenate([aux[ao[p]:ao[p + 1]] for p in range(len(d)) if owners[p] == r])
            local.append(W.max_sound_speed(a_r, sub))
        assert len(set(local)) > 1, local


HIER_WORKER = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1808_02638_b200 import binding, workloads as W
rank, world, idhex, name, out = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5], sys.argv[6]
wl = getattr(W, name)()
nlev = len(wl.levels)
q0s = W.hierarchy_ic(wl)
d = wl.levels[-1].descs
owners = binding.partition(d, world)
offs = W.level_offsets(d)
g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0, rank=rank, world=world,
                 nccl_id=bytes.fromhex(idhex), dist_level=nlev)
for L, (lv, q) in enumerate(zip(wl.levels, q0s), start=1):
    if L < nlev:
        g.set_level(L, lv.descs, q)
    else:
        g.set_level(L, lv.descs, np.concatenate([q[offs[p]:offs[p + 1]] for p in range(len(d)) if owners[p] == rank]))
dt = wl.dt0()
cfl = g.advance_hierarchy_n(0.0, dt, 3, update=True).tolist()
cfl.append(g.advance_hierarchy(3 * dt, dt, update=True))
for L in range(1, nlev + 1):
    np.save(out + f".L{L}.npy", g.read_level(L))
np.save(out + ".cfl.npy", np.array(cfl))
g.close()
'''


@pytest.mark.parametrize("world,name", [(2, "c2"), (3, "c2"), (2, "c3")])
def test_nccl_path_hierarchy_replicated_coarse_partitioned_finest(shim, tmp_path, world, name):
    """claw_config.dist_level through the library's NCCL path (stand-in NCCL,
    processes on one GPU): the native hierarchy driver exchanges the finest
    level's halo and, after its updating, the averaged coarse cells (grouped
    send/recv), and reduces the per-step CFLs once per call.  Every rank's
    coarse replicas and its own fine patches are bitwise the one-rank run."""
    env = dict(os.environ, CLAW_NCCL_LIB=shim)
    gen = subprocess.run([sys.executable, "-c",
                          "import sys; sys.path.insert(0, sys.argv[1]); "
                          "from paper_1808_02638_b200 import binding; print(binding.nccl_unique_id().hex())", ROOT],
                         env=env, capture_output=True, text=True, check=True)
    idhex = gen.stdout.strip().splitlines()[-1]
    script = tmp_path / "hworker.py"
    script.write_text(HIER_WORKER)
    procs = [subprocess.Popen([sys.executable, str(script), ROOT, str(r), str(world), idhex, name,
                               str(tmp_path / f"rank{r}")], env=env, stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for r in range(world)]
    outs = [p.communicate(timeout=600) for p in procs]
    for p, (so, se) in zip(procs, outs):
        assert p.returncode == 0, se[-3000:]
    wl = getattr(W, name)()
    nlev = len(wl.levels)
    ref = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0)
    for L, (lv, q) in enumerate(zip(wl.levels, W.hierarchy_ic(wl)), start=1):
        ref.set_level(L, lv.descs, q)
    dt = wl.dt0()
    cfl = ref.advance_hierarchy_n(0.0, dt, 3, update=True).tolist()
    cfl.append(ref.advance_hierarchy(3 * dt, dt, update=True))
    d = wl.levels[-1].descs
    owners = binding.partition(d, world)
    offs = W.level_offsets(d)
    for r in range(world):
        for L in range(1, nlev):
            assert np.array_equal(np.load(tmp_path / f"rank{r}.L{L}.npy"), ref.read_level(L)), (r, L)
        full = ref.read_level(nlev)
        mine = np.concatenate([full[offs[p]:offs[p + 1]] for p in range(len(d)) if owners[p] == r])
        assert np.array_equal(np.load(tmp_path / f"rank{r}.L{nlev}.npy"), mine), r
        assert np.load(tmp_path / f"rank{r}.cfl.npy").tolist() == cfl
    ref.close()
