#!/bin/bash
OUT=gpurun_out/r01_2v; mkdir -p $OUT
for tr in 8 16 32; do for sd in 0 1; do
  CLAW_SIDE=$sd timeout 600 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --tile-rows $tr > $OUT/c3_tr${tr}_side$sd.json 2>/dev/null
done; done
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('%-24s %.3f G/s  %.4f ms/step kernel %.4f' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], r['avg_launch_ms']))" 2>/dev/null; done
