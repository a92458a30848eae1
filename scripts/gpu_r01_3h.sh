#!/bin/bash
# grid kernel with x-neighbours from shared memory: full GPU suite, C5/C4 vs the shuffle variant
OUT=gpurun_out/r01_3h; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_all.log 2>&1; echo "rc=$?" >> $OUT/pytest_all.log
for rep in 1 2; do for v in "" build/variants/libclaw_nosmemx.so; do
  tag=$(basename "${v:-smemx}" .so)_$rep
  CLAW_LIB=$v timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_$tag.json 2>$OUT/c5_$tag.err
  CLAW_LIB=$v timeout 300 python bench.py --config c4 --steps 80 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c4_$tag.json 2>$OUT/c4_$tag.err
done; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_grid -s 2 -c 1 -o $OUT/ncu_c5 python scripts/prof_step.py --config c5 --steps 3 > $OUT/ncu_c5.log 2>&1
tail -3 $OUT/pytest_all.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('%-26s %.2f G/s  %.4f ms/step frac %.4f' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], r['frac']))"; done
