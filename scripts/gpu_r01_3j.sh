#!/bin/bash
# device summed-area table for the clusterer: regrid/paper GPU tests, regrid phase timing, paper bench x2
OUT=gpurun_out/r01_3j; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_regrid.py tests/test_gpu_paper.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
CLAW_TRACE_PLAN=1 timeout 600 python scripts/regrid_timing.py > $OUT/regrid.txt 2> $OUT/regrid_trace.txt
for rep in 1 2; do
  timeout 300 python bench.py --config paper --steps 40 --warmup 4 --no-cpu-baseline --no-e2e > $OUT/paper_$rep.json 2>$OUT/paper_$rep.err
done
tail -3 $OUT/pytest.log; cat $OUT/regrid.txt; grep -E "auto L|regrid L" $OUT/regrid_trace.txt | tail -14
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); c=d['config']
print('%-14s %.3f G/s  %.4f ms/step regrid %.2f ms x %d' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], c['regrid_ms_mean'], c['regrids']))"; done
