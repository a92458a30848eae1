"""Minimal driver for ncu: set up a workload and run a few steps."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1808_02638_b200 import binding, workloads as W
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--tile-rows", type=int, default=0)
ap.add_argument("--path", type=int, default=0)
a = ap.parse_args()
wl = {"c4": W.c4, "c5": W.c5, "c1": W.c1}[a.config]()
d = wl.levels[0].descs
g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0, tile_rows=a.tile_rows, path=a.path)
g.set_level(1, d, W.ring_ic(d))
dt = wl.dt0()
for n in range(a.steps):
    g.fill_ghost(1, n * dt)
    c = g.advance_level(1, dt)
print("cfl", c)
