#!/bin/bash
# smallest automatic tile height 4 vs 8 (CLAW_MIN_TH) on the latency-bound workloads
OUT=gpurun_out/r02_bm; mkdir -p $OUT
for i in 1 2; do
  for m in 8 4; do
    for c in c3 c2 c1; do CLAW_MIN_TH=$m timeout 600 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/${c}_m${m}_$i.json 2> $OUT/${c}_m${m}_$i.err; done
    CLAW_MIN_TH=$m timeout 600 python bench.py --config paper --steps 24 --warmup 8 --no-cpu-baseline --no-e2e > $OUT/paper_m${m}_$i.json 2> $OUT/paper_m${m}_$i.err
  done
done
CLAW_MIN_TH=4 timeout 900 python -m pytest tests/test_gpu_lane.py tests/test_gpu_parity.py tests/test_gpu_long.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
tail -n 2 $OUT/tests.log
for f in $OUT/*_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'ms_per_step', round(j['ms_per_step'],4))" 2>&1 | tail -1)"; done
