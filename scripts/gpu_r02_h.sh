#!/bin/bash
# grid kernel with interleaved (p,u) ring: bitwise tests, bench C5/C4/C3, ncu
OUT=gpurun_out/r02_h; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -x --durations=5 > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
timeout 600 python bench.py --steps 50 --warmup 5 > $OUT/bench_c5.json 2> $OUT/bench_c5.err
timeout 600 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 600 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_grid_kernel -s 3 -c 1 -o $OUT/ncu_grid_c5 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_grid.log 2>&1
python scripts/ncu_summary.py $OUT/ncu_grid_c5.ncu-rep $OUT/ncu_grid_c5.json 12884901888 > /dev/null 2>&1
tail -n 3 $OUT/gpu_all.log
for f in $OUT/bench_*.json; do echo "$f $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'ms/step', round(j['ms_per_step'],4), 'frac', j['roofline']['frac'], 'e2e', round(j['e2e']['value']/1e9,3))")"; done
python -c "import json; j=json.load(open('$OUT/ncu_grid_c5.json'))[0]; print({k: j[k] for k in ('time_ms','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active','stall_share','traffic_over_algorithmic')})"
