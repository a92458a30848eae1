#!/bin/bash
# lane kernel with an out-of-line segment resolver: lane tests, C2/C3/paper bench x2
OUT=gpurun_out/r01_3r; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_lane.py tests/test_gpu_paper.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for rep in 1 2; do
  timeout 300 python bench.py --config c2 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/c2_$rep.json 2>$OUT/c2_$rep.err
  timeout 300 python bench.py --config paper --steps 40 --warmup 4 --no-cpu-baseline --no-e2e > $OUT/paper_$rep.json 2>$OUT/paper_$rep.err
done
CLAW_LANE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_lane -s 20 -c 1 -o $OUT/ncu_paper_lane python scripts/prof_hier.py --config paper --steps 3 > $OUT/ncu_paper.log 2>&1
tail -2 $OUT/pytest.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); c=d['config']
print('%-14s %.3f G/s  %.4f ms/step regrid %s' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], c.get('regrid_ms_mean')))"; done
