#!/bin/bash
# parallel Berger-Rigoutsos subtrees: regrid/paper tests, paper bench x3 with trace
OUT=gpurun_out/r01_3p; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_regrid.py tests/test_gpu_paper.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for rep in 1 2 3; do
  CLAW_TRACE_PLAN=1 timeout 300 python bench.py --config paper --steps 40 --warmup 4 --no-cpu-baseline --no-e2e > $OUT/paper_$rep.json 2>$OUT/paper_$rep.err
done
tail -2 $OUT/pytest.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); c=d['config']
print('%-14s %.3f G/s  %.4f ms/step regrid %.2f ms x %d' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], c['regrid_ms_mean'], c['regrids']))"; done
grep -hE "\] (BR|sat\+d2h|nest-split|regrid|plan) " $OUT/paper_3.err | awk '{k=$1" "$2" "$3; a[k]+=$4; n[k]++} END {for (k in a) printf "%-22s mean %6.2f n=%d\n", k, a[k]/n[k], n[k]}' | sort
