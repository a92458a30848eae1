#!/bin/bash
OUT=gpurun_out/r01w; mkdir -p $OUT
for tr in 0 8 16 32 64; do
  timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --tile-rows $tr > $OUT/bench_c3_$tr.json 2>>$OUT/bench_err.log
  timeout 300 python bench.py --config c2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --tile-rows $tr > $OUT/bench_c2_$tr.json 2>>$OUT/bench_err.log
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_launch_c3.log 2>&1
for f in $OUT/bench_*.json; do echo $f; python -c "import json,sys; j=json.load(open('$f')); print(j['value']/1e9, j['ms_per_step'])"; done
