#!/bin/bash
# latency-bound hierarchies: occupancy variants x tile rows (C3, C2); paper workload line
OUT=gpurun_out/r02_i; mkdir -p $OUT
for v in base w20 w24; do
  if [ $v = base ]; then unset CLAW_LIB; else export CLAW_LIB=build/variants/libclaw_$v.so; fi
  for tr in 0 16 8; do
    timeout 300 python bench.py --config c3 --steps 100 --warmup 10 --tile-rows $tr --no-cpu-baseline --no-e2e > $OUT/c3_${v}_t$tr.json 2> $OUT/c3_${v}_t$tr.err
    timeout 300 python bench.py --config c2 --steps 200 --warmup 10 --tile-rows $tr --no-cpu-baseline --no-e2e > $OUT/c2_${v}_t$tr.json 2> $OUT/c2_${v}_t$tr.err
  done
done
unset CLAW_LIB
timeout 900 python bench.py --config paper --steps 24 --warmup 9 --no-cpu-baseline > $OUT/paper.json 2> $OUT/paper.err
for f in $OUT/*.json; do echo "$f $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'ms/step', round(j['ms_per_step'],4))")"; done
