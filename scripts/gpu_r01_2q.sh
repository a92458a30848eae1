#!/bin/bash
OUT=gpurun_out/r01_2q; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
timeout 300 python scripts/regrid_timing.py > $OUT/regrid_timing.txt 2>&1
timeout 600 python bench.py --config paper --steps 40 --warmup 5 > $OUT/paper.json 2> $OUT/paper.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/c5.json 2> $OUT/c5.err
tail -n 3 $OUT/gpu_all.log; cat $OUT/regrid_timing.txt
for f in $OUT/paper.json $OUT/c5.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); c=d['config']
print('%-12s %.3f G/s %.3f ms/step regrids %s mean %s e2e %s' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], c['regrids'], c['regrid_ms_mean'], (d.get('e2e') or {}).get('value')))"; done
