#!/bin/bash
# Wide grid kernel: parity tests, then bench lines C5/C4 wide vs narrow.
OUT=gpurun_out/r01_3b; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_parity.py tests/test_gpu_multirank.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
for w in 1 0; do
  CLAW_GRID_WIDE=$w timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_w$w.json 2>$OUT/c5_w$w.err
  CLAW_GRID_WIDE=$w timeout 300 python bench.py --config c4 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c4_w$w.json 2>$OUT/c4_w$w.err
done
tail -15 $OUT/pytest.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('%-14s %.2f G/s  %.4f ms/step frac %.4f' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], r['frac']))"; done
