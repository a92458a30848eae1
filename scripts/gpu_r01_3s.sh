#!/bin/bash
# grid kernel occupancy variants after the register cuts: 4 (128 regs), 5 (96), 6 (80, small spills) CTAs/SM
OUT=gpurun_out/r01_3s; mkdir -p $OUT
for rep in 1 2; do for v in "" build/variants/libclaw_spec5.so build/variants/libclaw_spec6.so; do
  tag=$(basename "${v:-spec4}" .so)_$rep
  CLAW_LIB=$v timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_$tag.json 2>$OUT/c5_$tag.err
  CLAW_LIB=$v timeout 300 python bench.py --config c4 --steps 80 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c4_$tag.json 2>$OUT/c4_$tag.err
done; done
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('%-26s %.2f G/s  %.4f ms/step frac %.4f' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], r['frac']))"; done
