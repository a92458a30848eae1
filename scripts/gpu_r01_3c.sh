#!/bin/bash
# Wide grid kernel: tests, occupancy variants, ncu of wide vs narrow (C5)
OUT=gpurun_out/r01_3c; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_wide.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
for v in "" build/variants/libclaw_w8.so; do
  tag=$(basename "${v:-default}" .so)
  CLAW_LIB=$v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_$tag.json 2>$OUT/c5_$tag.err
  CLAW_LIB=$v timeout 300 python bench.py --config c4 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c4_$tag.json 2>$OUT/c4_$tag.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_grid -s 2 -c 1 -o $OUT/ncu_c5_wide python scripts/prof_step.py --config c5 --steps 3 > $OUT/ncu_c5w.log 2>&1
CLAW_GRID_WIDE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_grid -s 2 -c 1 -o $OUT/ncu_c5_narrow python scripts/prof_step.py --config c5 --steps 3 > $OUT/ncu_c5n.log 2>&1
tail -5 $OUT/pytest.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('%-24s %.2f G/s  %.4f ms/step frac %.4f' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], r['frac']))"; done
