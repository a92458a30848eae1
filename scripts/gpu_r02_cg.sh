#!/bin/bash
# smallest automatic tile height 2 vs 4 on the latency-bound configs
OUT=gpurun_out/r02_cg; mkdir -p $OUT
CLAW_MIN_TH=2 timeout 900 python -m pytest tests/test_gpu_lane.py tests/test_gpu_parity.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
tail -n 2 $OUT/tests.log
for i in 1 2; do
  for m in 4 2; do
    for c in c1 c2 c3; do CLAW_MIN_TH=$m timeout 600 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/${c}_m${m}_$i.json 2> $OUT/${c}_m${m}_$i.err; done
  done
done
for f in $OUT/*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'ms_per_step', round(j['ms_per_step'],4))" 2>&1 | tail -1)"; done
