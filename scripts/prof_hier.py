"""Minimal driver for ncu on a multi-level workload (c2, c3, paper): build the
hierarchy (paper: by regridding), run a few coarse steps natively."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1808_02638_b200 import binding, workloads as W
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="paper")
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
wl = {"c2": W.c2, "c3": W.c3, "paper": W.paper}[a.config]()
g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0)
for L, (lev, q) in enumerate(zip(wl.levels, W.hierarchy_ic(wl)), start=1):
    g.set_level(L, lev.descs, q)
if wl.extra.get("ratios"):
    import bench
    dx1 = float(wl.levels[0].descs["dx"][0])
    for L in range(1, 1 + len(wl.extra["ratios"])):
        if L > 1:
            g.fill_ghost(L, 0.0)
        g.regrid_auto(L, *bench.regrid_params(wl, L, float(g.descs(L)["dx"][0]), dx1, 0.02))
dt = wl.dt0()
for n in range(a.steps):
    c = g.advance_hierarchy(n * dt, dt, update=True)
print("cfl", c, [len(g.descs(L)) for L in (1, 2, 3)])
