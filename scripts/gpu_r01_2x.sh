#!/bin/bash
OUT=gpurun_out/r01_2x; mkdir -p $OUT
for tr in 8 16 32; do
  timeout 600 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --tile-rows $tr > $OUT/c3_tr$tr.json 2>/dev/null
done
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('%-24s %.3f G/s  %.4f ms/step' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step']))" 2>/dev/null; done
