#!/bin/bash
# Halo-lane generic kernel with the fast issue path: tests, bench lines (lane forced on/off, auto)
OUT=gpurun_out/r01_3f; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_lane.py tests/test_gpu_side.py -x -q > $OUT/pytest_lane.log 2>&1; echo "rc=$?" >> $OUT/pytest_lane.log
for L in 1 0 auto; do
  if [ $L = auto ]; then unset CLAW_LANE; else export CLAW_LANE=$L; fi
  timeout 300 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/c3_l$L.json 2>$OUT/c3_l$L.err
  timeout 300 python bench.py --config c2 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/c2_l$L.json 2>$OUT/c2_l$L.err
  timeout 300 python bench.py --config c5 --path 1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5gen_l$L.json 2>$OUT/c5gen_l$L.err
  timeout 300 python bench.py --config paper --steps 24 --warmup 4 --no-cpu-baseline --no-e2e > $OUT/paper_l$L.json 2>$OUT/paper_l$L.err
done
unset CLAW_LANE
CLAW_LANE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_lane -s 2 -c 1 -o $OUT/ncu_c5gen_lane python scripts/prof_step.py --config c5 --path 1 --steps 3 > $OUT/ncu.log 2>&1
tail -3 $OUT/pytest_lane.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('%-18s %.3f G/s  %.4f ms/step frac %s' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], r.get('frac')))"; done
