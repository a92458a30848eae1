#!/bin/bash
OUT=gpurun_out/r01_2n; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
CLAW_TRACE_PLAN=1 timeout 600 python bench.py --config paper --steps 40 --warmup 5 > $OUT/paper.json 2> $OUT/paper.err
timeout 600 python bench.py --config c3 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --regrid 8 > $OUT/c3_regrid8.json 2> $OUT/c3_regrid8.err
tail -n 3 $OUT/gpu_all.log
grep -v "^\[plan" $OUT/paper.err | tail -n 24
for f in $OUT/paper.json $OUT/c3_regrid8.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); c=d['config']
print('%-18s %.3f G/s %.3f ms/step regrids %d mean %.2f ms patches %s e2e %s' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], c['regrids'], c['regrid_ms_mean'] or 0, c['patches_after'], (d.get('e2e') or {}).get('value')))"; done
