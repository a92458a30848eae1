#!/bin/bash
# one interpolation launch for all R substeps of a fine level: full GPU suite, C2/C3/paper x2, C3 timeline
OUT=gpurun_out/r01_4m; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_all.log 2>&1; echo "rc=$?" >> $OUT/pytest_all.log
for rep in 1 2; do for cfg in c2 c3 paper; do
  st=100; [ $cfg = paper ] && st=40
  timeout 300 python bench.py --config $cfg --steps $st --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${cfg}_$rep.json 2>$OUT/${cfg}_$rep.err
done; done
timeout 600 python scripts/trace_c3.py c3 > $OUT/trace.log 2>&1; cp gpurun_out/trace_c3.txt $OUT/ 2>/dev/null
tail -3 $OUT/pytest_all.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); c=d['config']
print('%-14s %.3f G/s  %.4f ms/step regrid %s' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], c.get('regrid_ms_mean')))"; done
grep -c interp $OUT/trace_c3.txt; tail -2 $OUT/trace.log
