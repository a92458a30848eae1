"""Per-rank step time of the multi-GPU band partition, measured one rank at a
time on ONE GPU ("Per-rank step time").

A context is created as rank r of N with the external exchange (claw_config
exchange = 1: no NCCL, no halo is moved -- the frame keeps its zeros), so the
GPU runs exactly the launches rank r runs on an N-GPU box: the interior-tile
launch, then the edge-tile launch (band mode splits every step in two so the
halo can land behind the interior tiles).  Nothing waits on another rank: this
times the per-rank compute only; the halo transfer and the per-call CFL
all-reduce are not in it.  Lines: N, rank, ms per step (CUDA events around K
batched steps), the two launches' mean times (profiled pass right after), and
the projected speed-up t(1) / t(N) for a strong-scaled level.

usage: python scripts/rank_time.py [c5|c5vc|c2|c3] [K] [N ...]

c2 / c3: multi-rank hierarchies (claw_config.dist_level = the finest level:
coarse levels replicated, the finest partitioned); ms per coarse step.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1808_02638_b200 import binding, workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
Ns = [int(x) for x in sys.argv[3:]] or [1, 2, 4, 8]
wl = {"c5vc": W.c5_layered, "c2": W.c2, "c3": W.c3}.get(cfg, W.c5)()
nlev = len(wl.levels)
d = wl.levels[-1].descs
aux = W.media_field(d) if cfg == "c5vc" else None
dt = wl.dt0() if aux is None else 0.9 * float(d["dx"][0]) / W.max_sound_speed(aux, d)
t1 = None
for N in Ns:
    owners = binding.partition(d, N)
    for r in sorted({0, N // 2}):
        g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0, rank=r, world=N,
                         exchange=1 if N > 1 else 0, dist_level=nlev if nlev > 1 else 0)
        for L, lv in enumerate(wl.levels, start=1):
            g.set_level(L, lv.descs)
        if aux is not None:
            g.set_aux(1, aux)
        cells = int((d["mx"].astype(np.int64) * d["my"])[owners == r].sum())
        t = 0.0
        g.advance_hierarchy_n(t, dt, 5, update=nlev > 1)
        t += 5 * dt
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        done = 0
        while done < K:
            k = min(10, K - done)
            g.advance_hierarchy_n(t, dt, k, update=nlev > 1)
            t += k * dt
            done += k
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        g.set_profiling(True)
        g.reset_stats()
        g.advance_hierarchy_n(t, dt, 10, update=nlev > 1)
        st = g.stats()
        g.set_profiling(False)
        if N == 1:
            t1 = ms
        line = {"cfg": cfg, "N": N, "rank": r, "cells": cells, "ms_per_step": ms,
                "step_kernel_ms_per_step": st["step_ms"] / 10, "launches_per_step": st["step_launches"] / 10,
                "G_cell_updates_per_s_rank": cells / ms / 1e6,
                "projected_speedup": (t1 / ms) if t1 else None}
        print(json.dumps(line), flush=True)
        g.close()
