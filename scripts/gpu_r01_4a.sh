#!/bin/bash
# auto tile rows at half a tile per resident warp: full GPU suite, C1/C2/C3/paper x2, C4/C5 once
OUT=gpurun_out/r01_4a; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_all.log 2>&1; echo "rc=$?" >> $OUT/pytest_all.log
for rep in 1 2; do for cfg in c1 c2 c3 paper; do
  st=100; [ $cfg = paper ] && st=40
  timeout 300 python bench.py --config $cfg --steps $st --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${cfg}_$rep.json 2>$OUT/${cfg}_$rep.err
done; done
timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5.json 2>$OUT/c5.err
timeout 300 python bench.py --config c4 --steps 80 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c4.json 2>$OUT/c4.err
tail -2 $OUT/pytest_all.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); c=d['config']
print('%-14s %.3f G/s  %.4f ms/step regrid %s' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], c.get('regrid_ms_mean')))"; done
