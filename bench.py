#!/usr/bin/env python
"""Benchmark of the batched AMR-level advance (arXiv 1808.02638 hot path) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5|c4|c3|c2|c1|paper|c5vc]
                    [--impl reference] [--no-cpu-baseline]

One "step" = one level step of the whole hot path over the workload:
claw_fill_ghost (same-level/BC ghosts are pulled inside the step kernel; for
N > 1 this is the NCCL halo exchange) + claw_advance_level (the fused sm_100a
step kernel, the device block->grid CFL max, the NCCL max all-reduce for N > 1
and the 8-byte CFL read-back).  Metric: fp64 cell-updates/s of the whole job
(all ranks), BASELINE.json's metric.  Default workload: configs[4] (C5,
16,384^2 cells as 65,536 patches of 64^2; fits one B200), partitioned over N
ranks (strong scaling).  Multi-level configs (c2, c3) count one coarse step
(1 + R1 + R1 R2 level advances) as a step.

Rank 0 prints ONE JSON line.  --impl reference times the CPU oracle (the only
"reference" this paper-only build has) on a bounded sample of the same
workload, on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1808_02638_b200 import workloads as W  # noqa: E402

LIMNAME = {0: "none", 1: "minmod", 2: "superbee", 3: "vanLeer", 4: "MC"}
BYTES_PER_CELL = 48  # algorithmic: read q^n (3 x fp64) + write q^{n+1} (3 x fp64)
BYTES_PER_CELL_VC = 64  # variable media: + read the cell's (Z, c) (2 x fp64)


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def workload(name: str) -> W.Workload:
    return {"c1": W.c1, "c2": W.c2, "c3": W.c3, "c4": W.c4, "c5": W.c5, "paper": W.paper,
            "c5vc": W.c5_layered}[name]()


def hierarchy_ratios(wl: W.Workload) -> list:
    """R_L between levels L and L+1 (fixed hierarchies: from the levels;
    dynamic ones, created by regridding: from the workload's extra)."""
    if wl.extra.get("ratios"):
        return list(wl.extra["ratios"])
    return [wl.levels[L].ratio for L in range(1, len(wl.levels))]


def regrid_params(wl: W.Workload, L: int, dxl: float, dx1: float, tol_arg: float):
    """(tol, buffer, cutoff, max_dim, min_dim, R) of the regrid of level L+1
    from level L (R18/R19)."""
    R = hierarchy_ratios(wl)
    e = wl.extra
    if e.get("ratios"):
        buf = int(e["buffer_coarse_cells"] * np.prod(R[:L - 1]))
        return e["tol_per_dx"] * dxl, buf, e["cutoff"], e["max_dim"], e["min_dim"], R[L - 1]
    return tol_arg * dxl / dx1, 2, 0.7, 32, 4, R[L - 1]


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clock, power and clock-event reasons sampled every 5 ms through NVML
    (nvidia-ml-py) while the timed region runs, so even a ~0.1 s region gets
    tens of samples; falls back to `nvidia-smi -lms 100`."""
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int, period_s: float = 0.005):
        self.device = device
        self.period = period_s
        self.rows = []       # (sm_mhz, max_mhz, power_w, reasons-set)
        self.proc = None
        self.thread = None
        self.stop_ev = threading.Event()
        self.source = None
        self.nv = None
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            uuid = str(torch.cuda.get_device_properties(device).uuid)
            self.h = nv.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            self.nv = nv
            self.source = f"nvml every {period_s * 1000:.0f} ms"
        except Exception:  # noqa: BLE001 -- any NVML problem: use nvidia-smi
            self.nv = None

    def _nvml_loop(self):
        nv = self.nv
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        while not self.stop_ev.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                bits = get_r(self.h)
                self.rows.append((float(sm), float(mx), pw, {k for k, b in self.BITS.items() if bits & b}))
            except Exception:  # noqa: BLE001
                pass
            self.stop_ev.wait(self.period)

    def start(self):
        if self.nv is not None:
            self.thread = threading.Thread(target=self._nvml_loop, daemon=True)
            self.thread.start()
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.source = "nvidia-smi -lms 100"
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._smi_loop, daemon=True)
        self.thread.start()

    def _smi_loop(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.proc.stdout:
            r = [x.strip() for x in line.split(",")]
            if len(r) >= 9:
                try:
                    self.rows.append((float(r[1]), float(r[2]), float(r[3]),
                                      {names[k] for k in range(4) if r[5 + k].lower() == "active"}))
                except ValueError:
                    pass

    def stop(self):
        self.stop_ev.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted(set().union(*(r[3] for r in self.rows))), "samples": len(self.rows),
                "power_w_max": max(r[2] for r in self.rows), "source": self.source}


# ---------------------------------------------------------------------------
# CPU oracle on a bounded sample (cpu_baseline / --impl reference)
# ---------------------------------------------------------------------------
def oracle_sample(wl: W.Workload, budget_s: float = 12.0, steps_cap: int | None = None, reflux: bool = False,
                  threads: int | None = None):
    """Time the oracle as it stands on a sub-level of the same workload shape
    (same patch size, same scheme) for ~budget_s of CPU work, with `threads`
    OpenMP threads over patches (default: every host core).  Returns
    (cell-updates/s, cores, description)."""
    import oracle
    d0 = wl.levels[0].descs
    mx, my = int(d0["mx"][0]), int(d0["my"][0])
    uniform = len(wl.levels) == 1 and not wl.extra.get("ratios") and (d0["mx"] == mx).all() and \
        (d0["my"] == my).all()
    cores = threads or host_cores()
    if uniform:
        side = max(1, min(int(math.sqrt(len(d0))), max(1, 1024 // mx)))  # ~1024^2 cells max
        dx = float(d0["dx"][0])
        dom = (-1.0, -1.0 + side * mx * dx, -1.0, -1.0 + side * my * dx)
        descs = W.uniform_level(side, side, mx, my, dom)
        q0 = W.ring_ic(descs)
        levels = [descs]
        desc = f"{side}x{side} patches of {mx}x{my} ({side*mx}x{side*my} cells) cut from {wl.name}"
    else:
        levels = [L.descs for L in wl.levels]
        desc = f"full {wl.name} hierarchy"
        q0 = None
    o = oracle.Oracle(wl.domain if not uniform else dom, wl.bc, wl.limiter, wl.order_trans, nthreads=cores,
                      reflux=reflux and not uniform)
    if uniform:
        o.set_level(1, levels[0], q0)
        if wl.extra.get("media"):
            o.set_aux(1, W.media_field(levels[0], wl.extra["media"]))
            desc += " (variable media)"
        cells = int((levels[0]["mx"].astype(np.int64) * levels[0]["my"]).sum())
        dt = wl.dt0()
        n, t0 = 0, time.perf_counter()
        while True:
            o.fill_ghost(1, n * dt)
            o.advance_level(1, dt)
            n += 1
            el = time.perf_counter() - t0
            if el >= budget_s or (steps_cap and n >= steps_cap):
                break
        return cells * n / el, cores, f"{desc}, {n} steps, {el:.1f} s"
    dyn = bool(wl.extra.get("ratios"))
    if dyn:  # the same dynamic workload on a 200^2 base (4 x 4 patches)
        wl = W.paper(n1=200, npx=4)
        o = oracle.Oracle(wl.domain, wl.bc, wl.limiter, wl.order_trans, nthreads=cores)
        desc = f"{wl.name} (base 200^2 sample of the 1000^2 workload), regrid every {wl.extra['regrid_every']}"
    for L, (lv, q) in enumerate(zip(wl.levels, W.hierarchy_ic(wl)), start=1):
        o.set_level(L, lv.descs, q)
    rat = hierarchy_ratios(wl)
    nlev = 1 + len(rat)
    dx1 = float(wl.levels[0].descs["dx"][0])
    counted = [0]

    def regrid(t):
        for L in range(1, nlev):
            if L > 1:
                o.fill_ghost(L, t)
            tol, buf, cut, mxd, mnd, R = regrid_params(wl, L, float(o.descs(L)["dx"][0]), dx1, 0.02)
            oracle.regrid_auto(o, L, tol, buf, cut, mxd, mnd, R)

    def bo(level, t, dt):
        o.fill_ghost(level, t)
        o.advance_level(level, dt)
        counted[0] += int((o.descs(level)["mx"].astype(np.int64) * o.descs(level)["my"]).sum())
        if level < nlev and len(o.descs(level + 1)):
            R = rat[level - 1]
            for k in range(R):
                bo(level + 1, t + k * dt / R, dt / R)
            o.update_level(level + 1)

    every = wl.extra.get("regrid_every", 0) if dyn else 0
    if dyn:
        regrid(0.0)
    dt = wl.dt0()
    n, t0 = 0, time.perf_counter()
    while True:
        bo(1, n * dt, dt)
        n += 1
        if every and n % every == 0:
            regrid(n * dt)
        el = time.perf_counter() - t0
        if el >= budget_s or (steps_cap and n >= steps_cap):
            break
    return counted[0] / el, cores, f"{desc}, {n} coarse steps (with updating), {el:.1f} s"


def mem_available_bytes() -> int:
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def oracle_workload_stepper(wl: W.Workload, cores: int, reflux: bool):
    """The oracle holding the WHOLE workload (C4/C5: every patch at full size,
    when the host has the memory; fixed hierarchies: every level), and a
    function that runs one of its steps (a level step of the uniform level, a
    Berger-Oliger coarse step with updating of a hierarchy).  Returns (step,
    cell-updates per step, description) or None when the full size does not
    fit the host memory."""
    import oracle
    d0 = wl.levels[0].descs
    if len(wl.levels) == 1:
        cells = int((d0["mx"].astype(np.int64) * d0["my"]).sum())
        media = wl.extra.get("media")
        need = (24 + (16 if media else 0)) * int(((d0["mx"].astype(np.int64) + 4) * (d0["my"] + 4)).sum()) + \
            (2 * 24 + (16 if media else 0)) * cells
        if need * 1.5 > mem_available_bytes():
            return None
        o = oracle.Oracle(wl.domain, wl.bc, wl.limiter, wl.order_trans, nthreads=cores)
        o.set_level(1, d0, W.ring_ic(d0))
        if media:
            o.set_aux(1, W.media_field(d0, media))
        dt = wl.dt0()
        n = [0]

        def step():
            o.fill_ghost(1, n[0] * dt)
            o.advance_level(1, dt)
            n[0] += 1
        return step, cells, f"the full {wl.name} level ({len(d0)} patches, {cells} cells), one level step per step"
    o = oracle.Oracle(wl.domain, wl.bc, wl.limiter, wl.order_trans, nthreads=cores, reflux=reflux)
    for L, (lv, q) in enumerate(zip(wl.levels, W.hierarchy_ic(wl)), start=1):
        o.set_level(L, lv.descs, q)
    rat = hierarchy_ratios(wl)
    nlev = 1 + len(rat)
    dt = wl.dt0()
    n = [0]

    def bo(level, t, dtl):
        o.fill_ghost(level, t)
        o.advance_level(level, dtl)
        if level < nlev:
            R = rat[level - 1]
            for k in range(R):
                bo(level + 1, t + k * dtl / R, dtl / R)
            o.update_level(level + 1)

    def step():
        bo(1, n[0] * dt, dt)
        n[0] += 1
    cells = sum(int((lv.descs["mx"].astype(np.int64) * lv.descs["my"]).sum()) * int(np.prod(rat[:L]))
                for L, lv in enumerate(wl.levels))
    return step, cells, f"the full {wl.name} hierarchy, one coarse step (with updating) per step"


def run_reference(args, rank):
    """The reference arm of this paper-only build: the CPU oracle as it stands,
    on the host cores, on the same workload.  Each step is one step of the
    WHOLE workload (C5: all 268 M cells) when the host memory holds it and K
    of them fit a few minutes; otherwise each step is a bounded sample of it
    (said in cpu_baseline.sample)."""
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    wl = workload(args.config)
    cores = host_cores()
    budget_s = 240.0
    t_setup = time.perf_counter()
    st = None if wl.extra.get("ratios") else oracle_workload_stepper(wl, cores, args.reflux)
    setup_s = time.perf_counter() - t_setup
    times = []
    if st is not None:
        step, cells, desc = st
        t0 = time.perf_counter()
        step()                                   # first warm-up step sizes the run
        first = time.perf_counter() - t0
        if first * (args.steps + max(args.warmup - 1, 0)) > budget_s:
            st = None                            # too slow for K full steps: bounded samples instead
            del step
        else:
            for _ in range(max(args.warmup - 1, 0)):
                step()
            for _ in range(args.steps):
                t0 = time.perf_counter()
                step()
                times.append(time.perf_counter() - t0)
            value = cells * len(times) / sum(times)
            ms_per_step = 1000.0 * sum(times) / len(times)
            desc = f"{desc}; {len(times)} timed steps after {args.warmup} warm-up, setup {setup_s:.1f} s"
    if st is None:
        vals, desc = [], ""
        for _ in range(args.warmup):
            oracle_sample(wl, budget_s=2.0, steps_cap=1, reflux=args.reflux)
        for _ in range(args.steps):
            v, cores, desc = oracle_sample(wl, budget_s=max(1.0, 60.0 / max(args.steps, 1)), steps_cap=None,
                                           reflux=args.reflux)
            vals.append(v)
        value = statistics.median(vals)
        cells = wl.levels[0].cells if len(wl.levels) == 1 else None
        # one step of the workload at the sampled rate (not a measured step)
        ms_per_step = 1000.0 * cells / value if cells else None
        desc = f"bounded samples per step: {desc} (median of {args.steps})"
    line = {"impl": "reference", "metric": "fp64 cell-updates/s", "value": value, "unit": "cell-updates/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl.name, "note": wl.note,
                       "conservation_fix": bool(args.reflux and len(wl.levels) > 1)},
            "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": cores, "kind": "oracle",
                             "sample": desc, "cpu": cpu_model()},
            "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` without a launcher: start N ranks of this same
    command through torch.distributed.run (one process per GPU, rendezvous on
    127.0.0.1); rank 0 prints the JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    print(f"[bench] spawning {n} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.run(cmd).returncode


# ---------------------------------------------------------------------------
# the GPU arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5", "paper", "c5vc"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--tile-rows", type=int, default=0)
    ap.add_argument("--path", type=int, default=0, help="0 auto (grid kernel for uniform levels), 1 generic")
    ap.add_argument("--reflux", action="store_true",
                    help="multi-level configs: conservation fix at coarse-fine interfaces (NEXT-2)")
    ap.add_argument("--regrid", type=int, default=-1,
                    help="multi-level configs: regrid every K coarse steps inside the timed region (NEXT-3; "
                         "claw_regrid_auto of levels 1..L-1, flag tol scaled by dx)")
    ap.add_argument("--regrid-tol", type=float, default=0.02)
    ap.add_argument("--batch", type=int, default=10,
                    help="fixed multi-level hierarchies: coarse steps per host synchronisation "
                         "(claw_advance_hierarchy_n; 1 = one claw_advance_hierarchy call per coarse step)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "host"],
                    help="host: TEST MODE -- halos through host memory over a gloo group "
                         "(claw exchange=1), ranks may share one GPU; never a bench number")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    world = env_int("WORLD_SIZE", 1)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but {world} rank(s) were launched (WORLD_SIZE); "
                         "launch N ranks with --gpus N, or omit the launcher and let --gpus N spawn them")
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        sys.exit(run_reference(args, rank))

    import torch
    import torch.distributed as dist

    from paper_1808_02638_b200 import binding

    host_x = args.exchange == "host" and world > 1
    # TEST MODE: CLAW_NCCL_LIB points libclaw at a stand-in NCCL that runs
    # between processes sharing one GPU (tests/nccl_shim); torch's plumbing
    # then uses gloo, since real NCCL refuses two ranks on one GPU
    shim_x = world > 1 and not host_x and bool(os.environ.get("CLAW_NCCL_LIB"))
    test_x = host_x or shim_x
    device = local_rank % max(1, torch.cuda.device_count()) if test_x else local_rank
    torch.cuda.set_device(device)
    if world > 1:
        if test_x:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    red_dev = "cpu" if test_x else "cuda"
    wl = workload(args.config)
    dyn = bool(wl.extra.get("ratios"))
    rat = hierarchy_ratios(wl)
    nlev = 1 + len(rat)
    if args.regrid < 0:
        args.regrid = wl.extra.get("regrid_every", 0) if dyn else 0
    if world > 1 and nlev > 1 and (dyn or args.regrid or args.reflux or args.exchange == "host"):
        raise SystemExit("multi-rank hierarchies: fixed hierarchies only (no regridding, no conservation fix, "
                         "NCCL exchange)")
    # multi-rank hierarchies: the coarse levels replicated, the finest
    # partitioned (claw_config.dist_level)
    dist_level = nlev if (world > 1 and nlev > 1) else 0

    # NCCL unique id for the library's own communicator (plumbing via torch)
    nccl_id = None
    if world > 1 and not host_x:
        obj = [binding.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    stream = torch.cuda.current_stream()
    g = binding.Claw(wl.domain, wl.bc, wl.limiter, wl.order_trans, device=device, rank=rank,
                     world=world, nccl_id=nccl_id, stream=stream.cuda_stream, tile_rows=args.tile_rows,
                     path=args.path, exchange=1 if host_x else 0, reflux=args.reflux and nlev > 1,
                     dist_level=dist_level)
    comm = None
    if world > 1:
        ci = g.comm_info()   # the communicator as NCCL reports it (None: external exchange)
        comm = {"rank": rank, "world": world, "cuda_device": device,
                "nccl_nranks": ci[0] if ci else None, "nccl_rank": ci[1] if ci else None,
                "nccl_cuda_device": ci[2] if ci else None}
        print(f"[bench] rank {rank}/{world} cuda:{device}: libclaw NCCL communicator "
              + (f"nranks={ci[0]} rank={ci[1]} cudaDev={ci[2]}" if ci else "none (external exchange)"),
              file=sys.stderr, flush=True)
        if ci and (ci[0] != world or ci[1] != rank):
            raise SystemExit(f"rank {rank}: NCCL communicator reports nranks={ci[0]} rank={ci[1]}")

    # inputs: host-side synthetic data of the workload's shape, uploaded once
    # through the API; pinned so the e2e leg measures the real H2D path
    host_q = []
    for L, lv in enumerate(wl.levels, start=1):
        owner = binding.partition(lv.descs, world) if (L == max(dist_level, 1)) else np.full(len(lv.descs), rank)
        mine = lv.descs[owner == rank]
        n = 3 * int((mine["mx"].astype(np.int64) * mine["my"]).sum())
        buf = torch.empty(n, dtype=torch.float64, pin_memory=True)
        W.ring_ic(mine, out=buf.numpy())
        g.set_level(L, lv.descs, buf)
        host_q.append(buf)
        if wl.extra.get("media"):
            # per-cell media of the whole level (problem description, set once;
            # every rank passes all of it and keeps its band + halo rows)
            g.set_aux(L, W.media_field(lv.descs, wl.extra["media"]))
    vc = bool(wl.extra.get("media"))
    bpc = BYTES_PER_CELL_VC if vc else BYTES_PER_CELL
    dt = wl.dt0()
    dx1 = float(wl.levels[0].descs["dx"][0])
    regrid_ms = []
    nstep = [0]

    def regrid(t):
        # every level L < nlev flags and re-creates L+1 (coarsest first)
        t0 = time.perf_counter()
        for L in range(1, nlev):
            if L > 1:
                g.fill_ghost(L, t)
            tol, buf, cut, mxd, mnd, R = regrid_params(wl, L, float(g.descs(L)["dx"][0]), dx1, args.regrid_tol)
            if g.regrid_auto(L, tol, buf, cut, mxd, mnd, R) == 0:
                break  # nothing flagged: level L+1 (and finer) removed; the next regrid may re-create them
        regrid_ms.append(1000.0 * (time.perf_counter() - t0))

    if dyn:
        regrid(0.0)  # the initial hierarchy from the initial data
    cells_owned = [g.level_owned(L)[1] for L in range(1, nlev + 1)]
    mult = [int(np.prod(rat[:L])) for L in range(nlev)]
    cells_per_step_rank = sum(c * m for c, m in zip(cells_owned, mult))
    total_cells_per_step = wl.levels[0].cells if nlev == 1 else cells_per_step_rank
    if dist_level:   # (replicated coarse levels count once in the whole-job total)
        total_cells_per_step = sum(int((lv.descs["mx"].astype(np.int64) * lv.descs["my"]).sum()) * m
                                   for lv, m in zip(wl.levels, mult))
    t_sim = [0.0]

    def host_exchange():
        # TEST MODE: the halo plan's cells through host memory and gloo
        reqs, inbox = [], {}
        for peer in range(world):
            if peer == rank:
                continue
            buf = g.halo_pack(1, peer)
            if buf.size:
                reqs.append(dist.isend(torch.from_numpy(buf), dst=peer))
            _, nrecv = g.debug_halo_counts(1, peer)
            if nrecv:
                inbox[peer] = torch.empty(3 * nrecv, dtype=torch.float64)
                reqs.append(dist.irecv(inbox[peer], src=peer))
        for r in reqs:
            r.wait()
        for peer, buf in inbox.items():
            g.halo_unpack(1, peer, buf.numpy())

    def step():
        t = t_sim[0]
        if nlev == 1:
            g.fill_ghost(1, t)
            if host_x:
                host_exchange()
            c = g.advance_level(1, dt)
            if host_x:
                cm = torch.tensor([c], dtype=torch.float64)
                dist.all_reduce(cm, op=dist.ReduceOp.MAX)
        else:
            # native subcycled coarse step with updating, one host sync
            g.advance_hierarchy(t, dt, update=True)
            nstep[0] += 1
            if args.regrid and nstep[0] % args.regrid == 0:
                regrid(t + dt)
        t_sim[0] = t + dt

    # fixed hierarchies and single levels (no regrid): K coarse steps per host
    # synchronisation (claw_advance_hierarchy_n; the per-step CFLs come back
    # together and are checked afterwards, DESIGN.md section 8 "K coarse steps
    # per host synchronisation")
    batch = not dyn and not args.regrid and args.batch > 1 and not host_x
    cfl_seen = []

    def steps(n):
        if not batch:
            for _ in range(n):
                step()
            return
        done = 0
        while done < n:
            k = min(args.batch, n - done)
            cfl_seen.extend(g.advance_hierarchy_n(t_sim[0], dt, k, update=True).tolist())
            t_sim[0] += k * dt
            done += k

    nwarm = max(args.warmup, 3) if args.warmup > 0 else 0
    if dyn and args.regrid and nwarm:
        # a dynamic hierarchy warms up through one regrid (its kernels, pool
        # chunks and host buffers), so the timed steps start in steady state
        nwarm = max(nwarm, args.regrid + 1)
    steps(nwarm)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timed region
    # (a bandwidth-bound level: CUDA events around every step launch, for the
    # roofline's per-launch time; a latency-bound step -- a hierarchy's
    # coarse step, ~30 event records, or C1's 40 us step -- would pay for
    # them, so its per-launch times come from a profiled pass of the same
    # length right after)
    prof_live = nlev == 1 and total_cells_per_step >= (1 << 24)
    g.reset_stats()
    g.set_profiling(prof_live)
    clocks = ClockSampler(device)
    clocks.start()
    time.sleep(0.3)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    regrid_ms.clear()
    ev0.record(stream)
    steps(args.steps)
    ev1.record(stream)
    barrier()
    clocks.stop()
    ms = ev0.elapsed_time(ev1)
    st = g.stats()
    share_ms = ms   # the time the step-kernel busy time is a share of
    if not prof_live:
        g.set_profiling(True)
        g.reset_stats()
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        steps(args.steps)
        p1.record(stream)
        torch.cuda.synchronize()
        stp = g.stats()
        for k in ("step_ms", "ghost_ms"):
            st[k] = stp[k]
        # (the profiled pass's own elapsed time: its per-launch events stretch
        # a latency-bound hierarchy, so the share is taken within that pass)
        share_ms = p0.elapsed_time(p1)
    if (args.regrid or dyn) and nlev > 1:
        # the hierarchy changes: count the cell-updates the library performed
        total_cells_per_step = st["cells_advanced"] / args.steps
        cells_per_step_rank = total_cells_per_step
    g.set_profiling(False)
    per_rank = None
    if world > 1:
        # every rank's device time of the K steps and its step-kernel busy
        # time; value uses the max over ranks
        mine = torch.tensor([ms, st["step_ms"]], dtype=torch.float64, device=red_dev)
        allr = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allr, mine)
        per_rank = {"ms": [float(x[0]) for x in allr], "step_kernel_busy_ms": [float(x[1]) for x in allr]}
        ms = max(per_rank["ms"])
        per_rank["max_ms"] = ms
        comms = [None] * world
        dist.all_gather_object(comms, comm)
        per_rank["comm"] = comms
    value = total_cells_per_step * args.steps / (ms / 1000.0)

    # ---- roofline of the dominant kernel (the fused step kernel)
    peak, peak_src = measured_peaks()
    # the step kernel's time per level advance (an advance is one launch, or
    # two -- interior and edge tiles -- when ranks overlap the halo exchange)
    advances = max(args.steps * sum(mult), 1)
    avg_ms = st["step_ms"] / advances
    bytes_per_launch = bpc * cells_per_step_rank / max(1, sum(mult))  # per level-launch mean
    if nlev == 1:
        bytes_per_launch = bpc * cells_owned[0]
    achieved = bytes_per_launch / (avg_ms / 1000.0) / 1e9 if avg_ms > 0 else None
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_step_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                pj = json.load(f)
            ent = pj.get(wl.name)
            if ent and world == 1 and nlev == 1:
                traffic = float(ent["dram_bytes_per_launch"])
        except (OSError, ValueError, KeyError):
            traffic = None
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "kernel": (f"step_vc_kernel<{LIMNAME[wl.limiter]},{wl.order_trans}>" if vc else
                       f"step_grid_kernel<{LIMNAME[wl.limiter]},{wl.order_trans}>" if g.level_mode(1) == "grid" and nlev == 1
                       else "level step kernels, mean per level launch (" +
                       ", ".join(f"L{L} {g.level_mode(L)}" for L in range(1, nlev + 1)) + ")" if nlev > 1
                       else f"step_kernel<{LIMNAME[wl.limiter]},{wl.order_trans},uniform>"),
            "bytes_per_cell": bpc,
            "bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_ms,
            "kernel_share_of_step": (st["step_ms"] / share_ms) if share_ms > 0 else None,
            "peak_source": peak_src,
            "nominal_8tbs_frac": (achieved / 8000.0) if achieved else None}

    # ---- e2e through the public API with host buffers (H2D + steps + D2H)
    e2e = None
    if not args.no_e2e and dyn:
        # dynamic hierarchy: H2D of the level-1 data, the initial regrid, K
        # coarse steps with their regrids, D2H of every level at the end.
        # The result buffers are the caller's: pinned, allocated before the
        # timed region with room for twice the levels of the device-timed run
        # (pinned allocation of hundreds of MB is not part of the method)
        cap = [2 * g.level_size(L) + 1024 for L in range(1, nlev + 1)]
        outs_cap = [torch.empty(c, dtype=torch.float64, pin_memory=True) for c in cap]
        barrier()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.reset_stats()
        g.set_level(1, wl.levels[0].descs, host_q[0])   # (re)starts the run at t = 0 from host data
        t_sim[0] = 0.0
        nstep[0] = 0
        regrid(0.0)
        for _ in range(args.steps):
            step()
        outs = []
        for L in range(1, nlev + 1):
            n = g.level_size(L)
            b = outs_cap[L - 1][:n] if n <= outs_cap[L - 1].numel() else torch.empty(n, dtype=torch.float64,
                                                                                     pin_memory=True)
            g.read_level(L, b)
            outs.append(b)
        e1.record(stream)
        barrier()
        ems = e0.elapsed_time(e1)
        wall = (time.perf_counter() - t0) * 1000.0
        e2e = {"value": g.stats()["cells_advanced"] / (ems / 1000.0), "unit": "cell-updates/s",
               "h2d_bytes_per_step": 8 * host_q[0].numel() / args.steps,
               "d2h_bytes_per_step": sum(8 * b.numel() for b in outs) / args.steps + 8,
               "ms": ems, "wall_ms": wall,
               "what": "set_level(1) from pinned host data + initial regrid + K x (coarse step + regrids every "
                       f"{args.regrid}) + read_level of every level (device->pinned host); cell-updates of the "
                       "timed run"}
    if not args.no_e2e and not dyn and not (args.regrid and nlev > 1):  # (regridding changes the level arrays)
        out_host = [torch.empty_like(b, pin_memory=True) for b in host_q]
        barrier()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for L, b in enumerate(host_q, start=1):
            g.write_level(L, b)
        steps(args.steps)
        for L, b in enumerate(out_host, start=1):
            g.read_level(L, b)
        e1.record(stream)
        barrier()
        ems = e0.elapsed_time(e1)
        wall = (time.perf_counter() - t0) * 1000.0
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=red_dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        state_bytes = sum(8 * b.numel() for b in host_q)
        e2e = {"value": total_cells_per_step * args.steps / (ems / 1000.0), "unit": "cell-updates/s",
               "h2d_bytes_per_step": state_bytes / args.steps + 8 * sum(mult),
               "d2h_bytes_per_step": state_bytes / args.steps + 8 * sum(mult),
               "ms": ems, "wall_ms": wall,
               "what": "write_level (pinned host->device) + K x (fill_ghost + advance_level -> 8-byte cfl"
                       + (f", read back {args.batch} at a time" if batch else "") + ") "
                       "+ read_level (device->pinned host), per rank, max over ranks"
                       + ("; the static medium is set once before (claw_set_aux, problem setup)" if vc else "")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        oracle.build()
        v, cores, desc = oracle_sample(wl, budget_s=12.0, reflux=args.reflux)
        v1, _, desc1 = oracle_sample(wl, budget_s=4.0, reflux=args.reflux, threads=1)
        cpu = {"value": v, "unit": "cell-updates/s", "cores": cores, "kind": "oracle", "sample": desc,
               "cpu": cpu_model(),
               "single_thread": {"value": v1, "cores": 1, "sample": desc1}}

    clk = clocks.summary()
    gpu_launches = st["step_launches"] + st["ghost_launches"]
    if rank == 0:
        if host_x:
            line_note = "TEST MODE --exchange host (halos through host memory): not a benchmark number"
        if shim_x:
            line_note = ("TEST MODE CLAW_NCCL_LIB (libclaw's NCCL path through a stand-in NCCL between processes "
                         "on one GPU): not a benchmark number")
        line = {"metric": "fp64 cell-updates/s", "value": value, "unit": "cell-updates/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": wl.name, "note": wl.note, "levels": nlev,
                           "patches": int(sum(len(lv.descs) for lv in wl.levels)),
                           "cells_per_step": total_cells_per_step, "limiter": wl.limiter, "order_trans": wl.order_trans,
                           "cfl": wl.cfl, "ic": "ring (Clawpack acoustics_2d_radial qinit)",
                           "medium": "layered, per-cell rho and K (workloads.LAYERS + inclusion)" if vc
                           else "homogeneous rho = K = 1",
                           "conservation_fix": bool(args.reflux and nlev > 1),
                           "regrid_every": args.regrid if nlev > 1 else 0,
                           "dynamic_hierarchy": dyn,
                           "warmup_steps_run": nwarm,
                           "limiter_name": {0: "none", 1: "minmod", 2: "superbee", 3: "van Leer", 4: "MC"}[wl.limiter],
                           "regrids": len(regrid_ms),
                           "coarse_steps_per_sync": args.batch if batch else 1,
                           "cfl_max_seen": max(cfl_seen) if cfl_seen else None,
                           "regrid_ms_mean": statistics.mean(regrid_ms) if regrid_ms else None,
                           "patches_after": [len(g.descs(L)) for L in range(1, nlev + 1)] if nlev > 1 else None,
                           "parallelism": (f"levels 1..{nlev - 1} replicated, level {nlev} patch-partitioned "
                                           f"over {world} rank(s); NCCL halo, update exchange, max all-reduce")
                           if dist_level else f"patch-partitioned over {world} rank(s), NCCL halo + max all-reduce"
                           if world > 1 else "single GPU",
                           "l2": "state per buffer exceeds L2 (126 MB); no flush needed"
                           if total_cells_per_step * 24 > 126e6 else "state fits L2 (latency-bound config)"},
                "roofline": roof, "clocks": clk, "e2e": e2e, "gpu_launches": gpu_launches,
                "per_gpu_value": value / world}
        if per_rank is not None:
            line["per_rank"] = per_rank
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if test_x:
            line["test_mode"] = line_note
        print(json.dumps(line), flush=True)
    g.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
