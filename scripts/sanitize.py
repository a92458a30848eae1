"""Small runs of every kernel family for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck); see scripts/gpu_sanitize.sh.

  grid     step_grid_kernel (dense): C1 and a reduced C4 (8x8 patches of 32^2,
           spanning tiles), both BCs
  generic  step_lane_kernel and step_kernel (+ side_kernel) on a ragged level
  hier     C3-shaped hierarchy (sparse-lattice grid kernel, interp_kernel,
           update kernels, reflux kernels) on a reduced C2 with reflux
  regrid   flag / dilate / sat / regrid kernels (claw_regrid_auto)
  vc       step_vc_kernel (variable media): a small grid, spanning tiles, the
           non-finite check
  band     band-split launches (interior rows [Y0+4, Y1-4), then the 4-row
           edge tiles) of the grid and vc kernels: 2 virtual ranks, external
           exchange
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1808_02638_b200 import binding, workloads as W  # noqa: E402

what = sys.argv[1:] or ["grid", "generic", "hier", "regrid", "vc", "band"]

if "grid" in what:
    for d, bc in ((W.c1().levels[0].descs, W.EXTRAP), (W.uniform_level(8, 8, 32, 32), W.PERIODIC)):
        if len(d) > 1:
            os.environ["CLAW_GRID_TH"] = "128"   # tiles spanning patch rows
        g = binding.Claw(W.DOMAIN, bc, 4, 2, device=0)
        os.environ.pop("CLAW_GRID_TH", None)
        g.set_level(1, d, W.random_ic(d, 1))
        for n in range(3):
            g.fill_ghost(1, 0.0)
            g.advance_level(1, 0.9 * float(d["dx"][0]))
        g.read_level(1)
        g.close()
    print("grid ok")

if "generic" in what:
    d = W.ragged_level(3, 70, 66, 40)
    for lane in ("1", "0"):
        os.environ["CLAW_LANE"] = lane
        g = binding.Claw(W.DOMAIN, W.EXTRAP, 3, 2, device=0)
        g.set_level(1, d, W.random_ic(d, 2))
        for n in range(3):
            g.fill_ghost(1, 0.0)
            g.advance_level(1, 0.8 * 2 / 70)
        g.read_level(1)
        g.close()
    os.environ.pop("CLAW_LANE")
    print("generic ok")

if "hier" in what:
    wl = W.c2()
    g = binding.Claw(wl.domain, wl.bc, 4, 2, device=0, reflux=True)
    for L, (lv, q) in enumerate(zip(wl.levels, W.hierarchy_ic(wl)), start=1):
        g.set_level(L, lv.descs, q)
    dt = wl.dt0()
    for n in range(2):
        g.advance_hierarchy(n * dt, dt, update=True)
    g.close()
    wl = W.c3()
    g = binding.Claw(wl.domain, wl.bc, 4, 2, device=0)
    for L, (lv, q) in enumerate(zip(wl.levels, W.hierarchy_ic(wl)), start=1):
        g.set_level(L, lv.descs, q)
    assert g.level_mode(3) == "sparse"
    g.advance_hierarchy(0.0, wl.dt0(), update=True)
    g.close()
    print("hier ok")

if "regrid" in what:
    wl = W.paper(n1=96, npx=2)
    g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=0)
    g.set_level(1, wl.levels[0].descs, W.hierarchy_ic(wl)[0])
    dx1 = float(wl.levels[0].descs["dx"][0])
    import bench
    for L in (1, 2):
        if L > 1:
            g.fill_ghost(L, 0.0)
        n = g.regrid_auto(L, *bench.regrid_params(wl, L, float(g.descs(L)["dx"][0]), dx1, 0.02))
        if n == 0:
            break
    g.advance_hierarchy(0.0, wl.dt0(), update=True)
    g.close()
    print("regrid ok")

if "vc" in what:
    for d, th in ((W.uniform_level(3, 2, 16, 12), None), (W.uniform_level(4, 8, 24, 16), "64")):
        if th:
            os.environ["CLAW_GRID_TH"] = th
        g = binding.Claw(W.DOMAIN, W.PERIODIC, 4, 2, device=0, check_finite=True)
        os.environ.pop("CLAW_GRID_TH", None)
        g.set_level(1, d, W.random_ic(d, 3))
        g.set_aux(1, W.random_media(d, 3))
        for n in range(3):
            g.fill_ghost(1, 0.0)
            g.advance_level(1, 0.3 * float(d["dy"][0]))
        g.read_level(1)
        g.close()
    print("vc ok")

if "band" in what:
    import numpy as np
    d = W.uniform_level(8, 8, 32, 32)
    offs = W.level_offsets(d)
    for media in (False, True):
        world = 2
        owners = binding.partition(d, world)
        q0 = W.random_ic(d, 4)
        ctxs = []
        for r in range(world):
            c = binding.Claw(W.DOMAIN, W.EXTRAP, 4, 2, device=0, rank=r, world=world, exchange=1)
            c.set_level(1, d, np.concatenate([q0[offs[p]:offs[p + 1]] for p in range(len(d)) if owners[p] == r]))
            if media:
                c.set_aux(1, W.random_media(d, 5))
            ctxs.append(c)
        for n in range(2):
            for c in ctxs:
                c.fill_ghost(1, 0.0)
            for r in range(world):
                for s_ in range(world):
                    if r != s_:
                        ctxs[s_].halo_unpack(1, r, ctxs[r].halo_pack(1, s_))
            for c in ctxs:
                c.advance_level(1, 0.3 * float(d["dx"][0]))
        for c in ctxs:
            c.read_level(1)
            c.close()
    print("band ok")
