#!/bin/bash
# RC 1 + L1 copies, CTA width 4 (default) vs 8 / 16, and 20 resident warps; GPU suite on the default
OUT=gpurun_out/r02_r; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
V="kw8 kw16 kw4r20"
for i in 1 2; do
  for v in base $V; do
    lib=build/variants/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
    CLAW_LIB=$lib timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_${v}_$i.json 2> $OUT/c5_${v}_$i.err
    CLAW_LIB=$lib timeout 600 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c4_${v}_$i.json 2> $OUT/c4_${v}_$i.err
  done
done
CLAW_ROWCOPY=0 timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_rc0.json 2> $OUT/c5_rc0.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_grid_kernel -s 3 -c 1 -o $OUT/ncu_grid_c5 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_grid.log 2>&1
python scripts/ncu_summary.py $OUT/ncu_grid_c5.ncu-rep $OUT/ncu_grid_c5.json 12884901888 > /dev/null 2>&1
tail -n 3 $OUT/gpu_all.log
for f in $OUT/c5_*.json $OUT/c4_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'frac', round(j['roofline']['frac'],4), 'launch_ms', round(j['roofline']['avg_launch_ms'],4))" 2>&1 | tail -1)"; done
python -c "import json; j=json.load(open('$OUT/ncu_grid_c5.json'))[0]; print({k: j[k] for k in ('time_ms','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','stall_share','traffic_over_algorithmic','l1tex__t_sector_hit_rate.pct')})"
