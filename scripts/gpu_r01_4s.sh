#!/bin/bash
# lane tiles capped at 32 rows (auto): full GPU suite, paper x3, C2/C3
OUT=gpurun_out/r01_4s; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_all.log 2>&1; echo "rc=$?" >> $OUT/pytest_all.log
for rep in 1 2 3; do timeout 300 python bench.py --config paper --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/paper_$rep.json 2>/dev/null; done
for cfg in c2 c3; do timeout 300 python bench.py --config $cfg --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/$cfg.json 2>/dev/null; done
tail -2 $OUT/pytest_all.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); c=d['config']
rg=c.get('regrid_ms_mean'); n=c.get('regrids') or 0
steps = (d['ms_per_step']*d['steps'] - (rg or 0)*n)/d['steps']
print('%-14s %.4f ms/step  steps-only %.4f  regrid %s' % ('$f'.split('/')[-1], d['ms_per_step'], steps, rg))"; done
