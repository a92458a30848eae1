#!/bin/bash
OUT=gpurun_out/r01e; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for v in 4_4 3_4 4_2 3_2; do
  for c in c5 c4; do
    CLAW_LIB=build/variants/libclaw_$v.so timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_${v}_$c.json 2>>$OUT/bench_err.log
  done
done
tail -3 $OUT/pytest_gpu.log
for f in $OUT/bench_*.json; do echo $f; python -c "import json,sys; j=json.load(open('$f')); print(j['value']/1e9, j['roofline']['frac'], j['ms_per_step'])"; done
