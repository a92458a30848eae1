"""Kernel timeline of C3 coarse steps via torch.profiler (CUPTI sees the
library's stream too): per-kernel durations and the gaps between them."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1808_02638_b200 import binding, workloads as W
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
wl = {"c2": W.c2, "c3": W.c3, "paper": W.paper}[cfg]()
g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0)
for L, (lev, q) in enumerate(zip(wl.levels, W.hierarchy_ic(wl)), start=1):
    g.set_level(L, lev.descs, q)
if wl.extra.get("ratios"):  # dynamic: the initial hierarchy by regridding
    import bench
    dx1 = float(wl.levels[0].descs["dx"][0])
    for L in range(1, 1 + len(wl.extra["ratios"])):
        if L > 1:
            g.fill_ghost(L, 0.0)
        g.regrid_auto(L, *bench.regrid_params(wl, L, float(g.descs(L)["dx"][0]), dx1, 0.02))
dt = wl.dt0()
t = 0.0
for n in range(5):
    g.advance_hierarchy(t, dt, update=True); t += dt
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for n in range(3):
        g.advance_hierarchy(t, dt, update=True); t += dt
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
rows = sorted([(e.time_range.start, e.time_range.end, e.name) for e in ev])
out = os.environ.get("OUT", "gpurun_out")
with open(os.path.join(out, f"trace_{cfg}.txt"), "w") as f:
    prev = None
    for s, e, nm in rows:
        gap = (s - prev) if prev is not None else 0
        f.write(f"{s:14.1f} dur {e-s:8.1f} gap {gap:8.1f}  {nm[:90]}\n")
        prev = e
tot = (rows[-1][1] - rows[0][0]) / 3 if rows else 0
busy = sum(e - s for s, e, _ in rows) / 3
print(json.dumps({"cfg": cfg, "us_per_coarse_step": tot, "busy_us": busy, "kernels_per_step": len(rows) / 3}))
