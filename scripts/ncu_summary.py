"""Summarise an ncu report (.ncu-rep) into a small JSON/markdown for profiles/.
usage: python scripts/ncu_summary.py REPORT.ncu-rep OUT.json [algorithmic_bytes]"""
import csv, io, json, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
alg = float(sys.argv[3]) if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second"]
res = []
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    ent = {k: d.get(k) for k in want}
    def f(k):
        try:
            return float(str(d.get(k, "nan")).replace(",", ""))
        except ValueError:
            return float("nan")
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    rb = f("dram__bytes_read.sum") * scale.get(u.get("dram__bytes_read.sum", "byte"), 1.0)
    wb = f("dram__bytes_write.sum") * scale.get(u.get("dram__bytes_write.sum", "byte"), 1.0)
    ent["dram_bytes_per_launch"] = rb + wb
    tms = f("gpu__time_duration.sum") * (1e-3 if u.get("gpu__time_duration.sum") == "us" else 1.0)
    ent["time_ms"] = tms
    ent["dram_GBps"] = (rb + wb) / (tms * 1e-3) / 1e9 if tms > 0 else None
    if alg:
        ent["algorithmic_bytes_per_launch"] = alg
        ent["traffic_over_algorithmic"] = (rb + wb) / alg
    stalls = {}
    for h, v in d.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v)
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    ent["stall_share"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]}
    res.append(ent)
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
