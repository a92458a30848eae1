#!/bin/bash
# batched hierarchy driver (C2/C3), fresh ncu of the C5 grid kernel with source, launch list
OUT=gpurun_out/r02_g; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_long.py -q -x -k "batched" > $OUT/batched.log 2>&1; echo "rc=$?" >> $OUT/batched.log
for b in 1 10 50; do
  timeout 600 python bench.py --config c3 --steps 100 --warmup 10 --batch $b --no-cpu-baseline > $OUT/bench_c3_b$b.json 2> $OUT/bench_c3_b$b.err
  timeout 600 python bench.py --config c2 --steps 200 --warmup 10 --batch $b --no-cpu-baseline > $OUT/bench_c2_b$b.json 2> $OUT/bench_c2_b$b.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_grid_kernel -s 3 -c 1 -o $OUT/ncu_grid_c5 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_grid.log 2>&1
python scripts/ncu_summary.py $OUT/ncu_grid_c5.ncu-rep $OUT/ncu_grid_c5.json 12884901888 > /dev/null 2>&1
tail -n 3 $OUT/batched.log
for f in $OUT/bench_*.json; do echo "$f $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'ms/step', round(j['ms_per_step'],4), 'e2e', round(j['e2e']['value']/1e9,3))")"; done
python -c "import json; j=json.load(open('$OUT/ncu_grid_c5.json'))[0]; print({k: j[k] for k in ('time_ms','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active','stall_share','traffic_over_algorithmic')})"
