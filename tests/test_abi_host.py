"""CPU tests of libclaw.so: it loads without a GPU, exports every symbol
include/claw.h declares, validates inputs, and its host planner resolves every
ghost cell exactly as the oracle's composite ghost rule does."""
import os
import re

import numpy as np
import pytest

import oracle
from paper_1808_02638_b200 import binding, workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "claw.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(claw_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_header_symbol():
    lib = binding.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(binding.EXPORTS)
    assert "sm_100a" in binding.version()


def test_library_is_built_for_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", binding.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def host_ctx(bc=W.EXTRAP, world=1, rank=0, limiter=4, domain=W.DOMAIN):
    return binding.Claw(domain, bc, limiter, 2, device=-1, rank=rank, world=world)


def code_field(descs):
    """Interior value = the cell's own donor code patch<<32 | lj<<16 | li
    (exact in fp64), so a ghost copy reveals its donor."""
    out = []
    for p, d in enumerate(descs):
        J, I = np.meshgrid(np.arange(d["my"]), np.arange(d["mx"]), indexing="ij")
        code = (p * 2.0 ** 32 + J * 2.0 ** 16 + I).astype(np.float64)
        out.append(np.stack([code, code, code]).ravel())
    return np.concatenate(out)


@pytest.mark.parametrize("bc", [W.EXTRAP, W.PERIODIC, (2, 2, 1, 1)])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_planner_ghost_sources_equal_oracle_composite_rule(bc, seed):
    d = W.ragged_level(seed, 26 + seed, 22, 8)
    g = host_ctx(bc)
    g.set_level(1, d)
    o = oracle.Oracle(W.DOMAIN, bc, 4, 2, nthreads=2)
    o.set_level(1, d, code_field(d))
    o.fill_ghost(1)
    for p in range(len(d)):
        src, _ = g.debug_ghost_sources(1, p)
        ref = o.read_padded(1, p)[0].astype(np.int64)
        assert np.array_equal(src, ref), p


def test_uniform_level_uses_few_rectangles_and_tiles():
    d = W.uniform_level(4, 4, 32, 32)
    g = host_ctx()
    g.set_level(1, d)
    n, cells, _ = g.level_owned(1)
    assert n == 16 and cells == 16 * 1024


@pytest.mark.parametrize("field,value", [("mx", 0), ("my", -1), ("mbc", 3), ("rho", 0.0), ("K", -1.0)])
def test_descriptor_validation(field, value):
    d = W.uniform_level(2, 2, 8, 8)
    d[field][1] = value
    g = host_ctx()
    with pytest.raises(binding.ClawError) as e:
        g.set_level(1, d)
    assert e.value.code == binding.CLAW_EINVAL
    assert "patch 1" in str(e.value)


def test_level_validation():
    g = host_ctx()
    d = W.uniform_level(2, 2, 8, 8)
    bad = d.copy(); bad["dx"][2] *= 2                    # dx differs within the level
    with pytest.raises(binding.ClawError):
        g.set_level(1, bad)
    bad = d.copy(); bad["xlower"][1] += 0.3 * d["dx"][1]   # off the grid
    with pytest.raises(binding.ClawError):
        g.set_level(1, bad)
    with pytest.raises(binding.ClawError):                 # does not tile
        g.set_level(1, d[:3])
    bad = d.copy(); bad["xlower"][1] = bad["xlower"][0]    # overlap
    with pytest.raises(binding.ClawError):
        g.set_level(1, bad)
    with pytest.raises(binding.ClawError) as e:            # level 2 before 1 on a fresh ctx
        host_ctx().set_level(2, d)
    assert e.value.code == binding.CLAW_ESTATE
    g.set_level(1, d)
    with pytest.raises(binding.ClawError) as e:
        g.fill_ghost(1, 0.0)
    assert e.value.code == binding.CLAW_ENODEV


def test_config_validation():
    for kw in (dict(limiter=7), dict(bc=(1, 2, 1, 1)), dict(bc=(3, 3, 1, 1))):
        args = dict(domain=W.DOMAIN, bc=W.EXTRAP, limiter=4)
        args.update(kw)
        with pytest.raises(binding.ClawError) as e:
            binding.Claw(args["domain"], args["bc"], args["limiter"], 2, device=-1)
        assert e.value.code == binding.CLAW_EINVAL


def test_fine_level_without_donor_is_enest():
    g = host_ctx()
    g.set_level(1, W.uniform_level(1, 1, 8, 8))
    # a fine patch (R=2) hugging the domain corner: every ghost has a donor
    fine = W.make_descs([0], [0], 4, 4, 2 / 16, 2 / 16)
    g.set_level(2, fine)
    src, _ = g.debug_ghost_sources(2, 0)
    assert (src == -1).sum() > 0          # coarse-interpolated ghosts exist


@pytest.mark.parametrize("world", [2, 3, 8])
def test_partition_uniform_grid_into_bands(world):
    """A uniform grid is cut into bands of whole patch rows (grid kernel per
    rank, halo = full rows); balanced to within one patch row."""
    d = W.uniform_level(16, 13, 16, 16)
    own = binding.partition(d, world)
    rows = own.reshape(13, 16)
    assert (rows == rows[:, :1]).all()                 # whole patch rows
    assert (np.diff(rows[:, 0]) >= 0).all()            # contiguous bands, ascending
    counts = np.bincount(rows[:, 0], minlength=world)
    assert counts.min() >= 13 // world and counts.max() <= 13 // world + 1
    assert np.array_equal(own, binding.partition(d, world))


@pytest.mark.parametrize("world", [2, 3, 8])
def test_partition_ragged_morton_balanced(world):
    d2 = W.ragged_level(5, 40, 36, 9)
    own2 = binding.partition(d2, world)
    cells = np.bincount(own2, weights=d2["mx"] * d2["my"], minlength=world)
    assert cells.max() <= cells.sum() / world + (d2["mx"] * d2["my"]).max()
    assert np.array_equal(own2, binding.partition(d2, world))


def test_nccl_stand_in_loads_through_claw_nccl_lib(tmp_path):
    """CPU: the test-only stand-in NCCL (tests/nccl_shim) compiles, exports the
    nine calls libclaw uses, and libclaw loads it through CLAW_NCCL_LIB (the
    unique id is the stand-in's); the GPU test runs the multi-process path."""
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    so = str(tmp_path / "libncclshim.so")
    subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-o", so, os.path.join(root, "tests", "nccl_shim", "ncclshim.c"),
                    "-ldl"], check=True)
    syms = subprocess.run(["nm", "-D", so], capture_output=True, text=True, check=True).stdout
    for f in ["GetUniqueId", "CommInitRank", "CommDestroy", "AllReduce", "Send", "Recv", "GroupStart", "GroupEnd",
              "GetErrorString"]:
        assert f" T nccl{f}" in syms, f
    code = ("import sys; sys.path.insert(0, sys.argv[1]); from paper_1808_02638_b200 import binding; "
            "print(binding.nccl_unique_id().split(b'\\0')[0].decode())")
    r = subprocess.run([sys.executable, "-c", code, root], env=dict(os.environ, CLAW_NCCL_LIB=so),
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().splitlines()[-1].startswith("/tmp/claw_ncclshim_")


def test_binding_rejects_bad_host_buffers_before_the_c_call():
    """every raw pointer the binding passes (set_level q0, write,
    write_level, read_level out=) is checked for dtype, contiguity, host
    residency and exact size; nothing reaches the C-ABI otherwise."""
    import torch
    d = W.uniform_level(2, 2, 4, 4)            # 4 patches of 4x4 -> 192 doubles
    n = 3 * 64
    g = host_ctx()
    # (numpy INPUTS of another dtype or stride are copied to float64 first;
    # torch tensors are never converted, and outputs never)
    bad = [np.zeros(n - 1), np.zeros(n + 3), np.zeros((n + 1, 2), np.float32)[:, 0],
           torch.zeros(n, dtype=torch.float32), torch.zeros(2 * n, dtype=torch.float64)[::2],
           torch.zeros(n - 1, dtype=torch.float64), [0.0] * (n - 1)]
    for q in bad:
        with pytest.raises(binding.ClawError) as e:
            g.set_level(1, d, q)
        assert e.value.code == binding.CLAW_EINVAL, q
    for out in (np.broadcast_to(np.zeros(1), (8,)), np.zeros(8, np.float32), np.zeros(16)[::2], np.zeros(7)):
        with pytest.raises(binding.ClawError) as e:  # output buffers: read-only, float32, strided, short
            binding._host_f64(out, 8, "out", writable=True)
        assert e.value.code == binding.CLAW_EINVAL
    for q in (np.zeros(n), torch.zeros(n, dtype=torch.float64)):
        assert binding._host_f64(q, n, "ok") is not None


def test_set_aux_validation_host_only():
    """claw_set_aux (variable media, R20): a uniform single-rank grid
    level only, positive finite rho / K, single-level afterwards."""
    d = W.uniform_level(2, 2, 8, 8)
    g = host_ctx()
    g.set_level(1, d)
    assert g.level_mode(1) == "grid"
    aux = W.random_media(d, 1)
    bad = aux.copy()
    bad[70] = -1.0
    with pytest.raises(binding.ClawError) as e:
        g.set_aux(1, bad)
    assert e.value.code == binding.CLAW_EINVAL and "rho" in str(e.value) or "K" in str(e.value)
    bad[70] = np.inf
    with pytest.raises(binding.ClawError):
        g.set_aux(1, bad)
    with pytest.raises(binding.ClawError):
        g.set_aux(1, aux[:-1])                 # wrong size (binding check)
    g.set_aux(1, aux)
    with pytest.raises(binding.ClawError) as e:  # no finer level under variable media
        g.set_level(2, W.make_descs([4], [4], 8, 8, 2 / 32, 2 / 32))
    assert e.value.code == binding.CLAW_EINVAL
    g.close()
    r = host_ctx()
    rd = W.ragged_level(3, 20, 18, 7)
    r.set_level(1, rd)
    with pytest.raises(binding.ClawError) as e:  # not a uniform grid
        r.set_aux(1, W.random_media(rd, 2))
    assert e.value.code == binding.CLAW_EINVAL
    r.close()


@pytest.mark.parametrize("name,world", [("c2", 2), ("c2", 3), ("c3", 2), ("c3", 4)])
def test_dist_level_update_exchange_plans_agree(name, world):
    """claw_config.dist_level (host-only contexts, one per rank): the coarse
    levels are replicated (every rank owns every patch), the finest is
    partitioned as claw_partition says; the update exchange lists agree
    pairwise (what rank r sends is what every other rank expects from r), and
    together they cover every coarse cell the finest level averages, once
    (the rectangles of the one-rank plan)."""
    wl = getattr(W, name)()
    nlev = len(wl.levels)
    ctxs = []
    for r in range(world):
        c = binding.Claw(wl.domain, wl.bc, 4, 2, device=-1, rank=r, world=world, exchange=1, dist_level=nlev)
        for L, lv in enumerate(wl.levels, start=1):
            c.set_level(L, lv.descs)
        ctxs.append(c)
    owners = binding.partition(wl.levels[-1].descs, world)
    for r, c in enumerate(ctxs):
        for L in range(1, nlev):
            assert [c.owner(L, p) for p in range(len(wl.levels[L - 1].descs))] == [r] * len(wl.levels[L - 1].descs)
        assert [c.owner(nlev, p) for p in range(len(owners))] == list(owners)
    sends = [c.debug_update_counts(nlev, r)[0] for r, c in enumerate(ctxs)]
    for s, cs in enumerate(ctxs):
        for r in range(world):
            if r != s:
                assert cs.debug_update_counts(nlev, r)[1] == sends[r]
    # the averaged coarse cells: every coarse cell whose R x R children are on the finest level
    R = wl.levels[-1].ratio
    fine = wl.levels[-1].descs
    cover = set()
    for d in fine:
        i0 = int(round((d["xlower"] - wl.domain[0]) / d["dx"]))
        j0 = int(round((d["ylower"] - wl.domain[2]) / d["dy"]))
        for J in range(j0 // R, (j0 + int(d["my"])) // R):
            for I in range(i0 // R, (i0 + int(d["mx"])) // R):
                cover.add((I, J))
    assert sum(sends) == len(cover)
    for c in ctxs:
        c.close()
