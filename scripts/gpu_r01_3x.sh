#!/bin/bash
# lane tiles also for latency-bound levels (lane tiles fit one wave): tests, C2/C3/paper x2
OUT=gpurun_out/r01_3x; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_all.log 2>&1; echo "rc=$?" >> $OUT/pytest_all.log
for rep in 1 2; do
  timeout 300 python bench.py --config c2 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/c2_$rep.json 2>$OUT/c2_$rep.err
  timeout 300 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/c3_$rep.json 2>$OUT/c3_$rep.err
  timeout 300 python bench.py --config paper --steps 40 --warmup 4 --no-cpu-baseline --no-e2e > $OUT/paper_$rep.json 2>$OUT/paper_$rep.err
done
tail -2 $OUT/pytest_all.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); c=d['config']
print('%-14s %.3f G/s  %.4f ms/step regrid %s' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], c.get('regrid_ms_mean')))"; done
