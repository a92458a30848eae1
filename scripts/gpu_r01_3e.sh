#!/bin/bash
# Halo-lane generic kernel: bitwise tests vs the side-pass kernel, full GPU suite, bench lines C3/paper/C5 forced generic
OUT=gpurun_out/r01_3e; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_lane.py -x -q > $OUT/pytest_lane.log 2>&1; echo "rc=$?" >> $OUT/pytest_lane.log
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_all.log 2>&1; echo "rc=$?" >> $OUT/pytest_all.log
for L in 1 0; do
  CLAW_LANE=$L timeout 300 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/c3_l$L.json 2>$OUT/c3_l$L.err
  CLAW_LANE=$L timeout 300 python bench.py --config c5 --path 1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5gen_l$L.json 2>$OUT/c5gen_l$L.err
  CLAW_LANE=$L timeout 300 python bench.py --config paper --steps 24 --warmup 4 --no-cpu-baseline --no-e2e > $OUT/paper_l$L.json 2>$OUT/paper_l$L.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_lane -s 2 -c 1 -o $OUT/ncu_c5gen_lane python scripts/prof_step.py --config c5 --path 1 --steps 3 > $OUT/ncu.log 2>&1
tail -3 $OUT/pytest_lane.log; tail -3 $OUT/pytest_all.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('%-18s %.3f G/s  %.4f ms/step frac %s' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], r.get('frac')))"; done
