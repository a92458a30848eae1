#!/bin/bash
# grid kernel: keep p, u of the x-swept row (2 LDS fewer per row) vs re-read
OUT=gpurun_out/r01_4k; mkdir -p $OUT
for rep in 1 2; do for v in "" build/variants/libclaw_keep1.so; do
  tag=$(basename "${v:-keep0}" .so)_$rep
  CLAW_LIB=$v timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_$tag.json 2>$OUT/c5_$tag.err
  CLAW_LIB=$v timeout 300 python bench.py --config c4 --steps 80 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c4_$tag.json 2>$OUT/c4_$tag.err
done; done
CLAW_LIB=build/variants/libclaw_keep1.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py -q -x -k "grid or wide or c5 or c4" > $OUT/pytest_keep1.log 2>&1; echo "rc=$?" >> $OUT/pytest_keep1.log
tail -2 $OUT/pytest_keep1.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('%-26s %.2f G/s  %.4f ms/step frac %.4f' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], r['frac']))"; done
