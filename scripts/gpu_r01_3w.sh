#!/bin/bash
# updating as a flat chunk list + exact power-of-two mean: full GPU suite, C3/C2/paper bench, trace
OUT=gpurun_out/r01_3w; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_all.log 2>&1; echo "rc=$?" >> $OUT/pytest_all.log
for rep in 1 2; do
  timeout 300 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/c3_$rep.json 2>$OUT/c3_$rep.err
  timeout 300 python bench.py --config paper --steps 40 --warmup 4 --no-cpu-baseline --no-e2e > $OUT/paper_$rep.json 2>$OUT/paper_$rep.err
done
timeout 600 python scripts/trace_c3.py paper > $OUT/trace_paper.log 2>&1; cp gpurun_out/trace_paper.txt $OUT/ 2>/dev/null
tail -2 $OUT/pytest_all.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); c=d['config']
print('%-14s %.3f G/s  %.4f ms/step regrid %s' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], c.get('regrid_ms_mean')))"; done
grep update_rect $OUT/trace_paper.txt | head -4
