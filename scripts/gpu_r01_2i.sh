#!/bin/bash
# occupancy variants of the specialised grid kernel (MINB_SPEC 4/5/6) on C5 and C4
OUT=gpurun_out/r01_2i; mkdir -p $OUT
V=paper_1808_02638_b200/build/variants
for rep in 1 2; do
for v in base spec5 spec6; do
  if [ $v = base ]; then L=paper_1808_02638_b200/libclaw.so; else L=$V/libclaw_$v.so; fi
  for cfg in c5 c4; do
    CLAW_LIB=$L timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $OUT/${cfg}_${v}_$rep.json 2>/dev/null
  done
done
done
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('%-40s %.2f G/s  kernel %.4f ms  frac %.3f' % ('$f'.split('/')[-1], d['value']/1e9, r['avg_launch_ms'], r['frac']))"; done
