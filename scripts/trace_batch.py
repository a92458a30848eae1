"""Kernel timeline of K coarse steps queued by claw_advance_hierarchy_n
(one host synchronisation) via torch.profiler: per-kernel durations, gaps,
GPU busy vs elapsed per coarse step, and the host time of the call."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1808_02638_b200 import binding, workloads as W
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
wl = {"c2": W.c2, "c3": W.c3}[cfg]()
g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0)
for L, (lev, q) in enumerate(zip(wl.levels, W.hierarchy_ic(wl)), start=1):
    g.set_level(L, lev.descs, q)
dt = wl.dt0()
t = 0.0
for n in range(3):
    g.advance_hierarchy_n(t, dt, K, update=True); t += K * dt
torch.cuda.synchronize()
t0 = time.perf_counter()
for n in range(3):
    g.advance_hierarchy_n(t, dt, K, update=True); t += K * dt
wall = (time.perf_counter() - t0) / (3 * K)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    g.advance_hierarchy_n(t, dt, K, update=True); t += K * dt
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
rows = sorted([(e.time_range.start, e.time_range.end, e.name) for e in ev])
out = os.environ.get("OUT", "gpurun_out")
with open(os.path.join(out, f"trace_batch_{cfg}.txt"), "w") as f:
    prev = None
    for s, e, nm in rows:
        gap = (s - prev) if prev is not None else 0
        f.write(f"{s:14.1f} dur {e-s:8.1f} gap {gap:8.1f}  {nm[:90]}\n")
        prev = e
tot = (rows[-1][1] - rows[0][0]) / K if rows else 0
busy = sum(e - s for s, e, _ in rows) / K
print(json.dumps({"cfg": cfg, "K": K, "wall_us_per_coarse_step_unprofiled": wall * 1e6,
                  "us_per_coarse_step": tot, "busy_us": busy, "kernels_per_step": len(rows) / K}))
