#!/bin/bash
OUT=gpurun_out/r01_3z; mkdir -p $OUT; CFG=${CFG:-c2}
for tr in 0 8 16 32 64; do
  timeout 300 python bench.py --config $CFG --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --tile-rows $tr > $OUT/${CFG}_tr$tr.json 2>/dev/null
done
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('%-14s %.3f G/s  %.4f ms/step' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step']))"; done
