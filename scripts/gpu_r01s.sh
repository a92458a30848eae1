#!/bin/bash
OUT=gpurun_out/r01s; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for c in c5 c4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_grid_$c.json 2>>$OUT/bench_err.log
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --path 1 > $OUT/bench_gen_$c.json 2>>$OUT/bench_err.log
done
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_c3.json 2>>$OUT/bench_err.log
tail -3 $OUT/pytest_gpu.log
for f in $OUT/bench_*.json; do echo $f; python -c "import json,sys; j=json.load(open('$f')); print(j['value']/1e9, j['roofline']['frac'], j['ms_per_step'])"; done
