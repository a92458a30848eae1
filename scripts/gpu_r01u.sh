#!/bin/bash
OUT=gpurun_out/r01u; mkdir -p $OUT
for c in c5 c4; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_base_$c.json 2>>$OUT/bench_err.log
  for v in 3_8 4_16 3_16; do
    CLAW_LIB=build/variants/libclaw_$v.so timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_${v}_$c.json 2>>$OUT/bench_err.log
  done
done
for f in $OUT/bench_*.json; do echo $f; python -c "import json,sys; j=json.load(open('$f')); print(j['value']/1e9, j['roofline']['frac'], j['ms_per_step'])"; done
