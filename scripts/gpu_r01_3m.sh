#!/bin/bash
# persistent host worker pool: full GPU suite, paper bench x3 with phase trace
OUT=gpurun_out/r01_3m; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_all.log 2>&1; echo "rc=$?" >> $OUT/pytest_all.log
for rep in 1 2 3; do
  CLAW_TRACE_PLAN=1 timeout 300 python bench.py --config paper --steps 40 --warmup 4 --no-cpu-baseline --no-e2e > $OUT/paper_$rep.json 2>$OUT/paper_$rep.err
done
tail -2 $OUT/pytest_all.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); c=d['config']
print('%-14s %.3f G/s  %.4f ms/step regrid %.2f ms x %d' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], c['regrid_ms_mean'], c['regrids']))"; done
for f in $OUT/*.err; do echo "== $f"; grep -E "\] [a-z-]+ +[0-9.]+ ms" $f | awk '{k=$1" "$2" "$3; a[k]+=$4; n[k]++; if ($4>m[k]) m[k]=$4} END {for (k in a) printf "%-24s mean %6.2f max %6.2f n=%d\n", k, a[k]/n[k], m[k], n[k]}' | sort; done
