#!/bin/bash
OUT=gpurun_out/r01j; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for c in c5 c4; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_def_$c.json 2>>$OUT/bench_err.log
  for v in 3_4; do
    CLAW_LIB=build/variants/libclaw_$v.so timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_${v}_$c.json 2>>$OUT/bench_err.log
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_ -s 2 -c 1 -o $OUT/prof_c5 python scripts/prof_step.py --config c5 --steps 3 > $OUT/ncu_c5.log 2>&1
tail -3 $OUT/pytest_gpu.log
for f in $OUT/bench_*.json; do echo $f; python -c "import json,sys; j=json.load(open('$f')); print(j['value']/1e9, j['roofline']['frac'], j['ms_per_step'])"; done
