#!/bin/bash
# GPU suite after the boundary / vc fixes; bench C5, C4, c5vc; occupancy variants of the grid kernel; vc ncu
OUT=gpurun_out/r02_f; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
for v in base w20 w24; do
  if [ $v = base ]; then export -n CLAW_LIB; unset CLAW_LIB; else export CLAW_LIB=build/variants/libclaw_$v.so; fi
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/bench_c5_$v.json 2> $OUT/bench_c5_$v.err
  timeout 600 python bench.py --config c4 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/bench_c4_$v.json 2> $OUT/bench_c4_$v.err
done
unset CLAW_LIB
timeout 600 python bench.py --config c5vc --steps 30 --warmup 5 --no-cpu-baseline > $OUT/bench_c5vc.json 2> $OUT/bench_c5vc.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_vc_kernel -s 2 -c 1 -o $OUT/ncu_vc_c5 -f python bench.py --config c5vc --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_vc.log 2>&1
python scripts/ncu_summary.py $OUT/ncu_vc_c5.ncu-rep $OUT/ncu_vc_c5.json 17179869184 > /dev/null 2>&1
tail -n 4 $OUT/gpu_all.log
for f in $OUT/bench_*.json; do echo "$f $(python -c "import json,sys; j=json.load(open('$f')); print(j['value']/1e9, j['roofline']['frac'], j['roofline']['avg_launch_ms'])")"; done
python -c "import json; j=json.load(open('$OUT/ncu_vc_c5.json'))[0]; print({k: j[k] for k in ('time_ms','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active','stall_share','traffic_over_algorithmic')})"
