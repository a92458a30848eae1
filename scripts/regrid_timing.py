"""Per-call timing of the dynamic paper workload's regrids (host wall clock)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1808_02638_b200 import binding, workloads as W
import bench
wl = W.paper()
g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0)
d1 = wl.levels[0].descs
g.set_level(1, d1, W.ring_ic(d1))
dx1 = float(d1["dx"][0])
def regrid(t):
    out = []
    for L in (1, 2):
        t0 = time.perf_counter()
        if L > 1:
            g.fill_ghost(L, t)
        t1 = time.perf_counter()
        p = bench.regrid_params(wl, L, float(g.descs(L)["dx"][0]), dx1, 0.02)
        t2 = time.perf_counter()
        g.regrid_auto(L, *p)
        t3 = time.perf_counter()
        out.append((round(1e3 * (t1 - t0), 2), round(1e3 * (t2 - t1), 2), round(1e3 * (t3 - t2), 2)))
    return out
print("init", regrid(0.0), binding.pool_stats())
dt = wl.dt0()
for n in range(48):
    t0 = time.perf_counter()
    g.advance_hierarchy(n * dt, dt, update=True)
    ts = 1e3 * (time.perf_counter() - t0)
    if (n + 1) % 8 == 0:
        print("step %.2f ms" % ts, "regrid", regrid((n + 1) * dt), binding.pool_stats())
