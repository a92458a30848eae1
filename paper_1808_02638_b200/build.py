"""In-tree build of libclaw.so for sm_100a (nvcc; cudart static; NCCL dlopen'ed)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libclaw.so")
SOURCES = [os.path.join(PKG, "csrc", "claw_kernels.cu"), os.path.join(PKG, "csrc", "claw_host.cpp")]
HEADERS = [os.path.join(PKG, "csrc", "claw_internal.h"), os.path.join(PKG, "csrc", "claw_vc.cuh"),
           os.path.join(ROOT, "include", "claw.h")]

NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-shared", "-Xptxas", "-warn-spills"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in SOURCES + HEADERS + [__file__])


def build(force: bool = False, verbose: bool = False, defs=(), out: str | None = None) -> str:
    """Compile every source to an object in parallel (nvcc -c), then link.
    defs / out: tuning variants (-D knobs) linked to another path."""
    lib = out or LIB
    if not force and out is None and not defs and not stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    odir = os.path.join(PKG, "build", "v_" + "_".join(d.lstrip("-D") for d in defs)) if defs else \
        os.path.join(PKG, "build")
    os.makedirs(odir, exist_ok=True)
    cflags = [f for f in NVCC_FLAGS if f != "-shared"]
    jobs = []
    # the kernels file is compiled once per wave limiter (-DCLAW_LIM=k: the
    # step / reflux template instances of that limiter) plus once for the rest
    units = [(src, []) for src in SOURCES] + [(SOURCES[0], [f"-DCLAW_LIM={k}"]) for k in range(5)]
    for src, dfs in units:
        tag = dfs[0].split("=")[1] if dfs else ""
        obj = os.path.join(odir, os.path.basename(src) + (f".lim{tag}" if tag else "") + ".o")
        jobs.append((obj, [nvcc(), *cflags, *dfs, *defs, "-I", os.path.join(ROOT, "include"), "-c", "-o", obj,
                           src]))
    if verbose:
        for _, cmd in jobs:
            print(" ".join(cmd), file=sys.stderr)
    with ThreadPoolExecutor(len(jobs)) as ex:
        for r in ex.map(lambda j: subprocess.run(j[1]), jobs):
            if r.returncode:
                raise subprocess.CalledProcessError(r.returncode, r.args)
    link = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", lib,
            *[o for o, _ in jobs], "-ldl"]
    if verbose:
        print(" ".join(link), file=sys.stderr)
    subprocess.run(link, check=True)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
