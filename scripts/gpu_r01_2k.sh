#!/bin/bash
OUT=gpurun_out/r01_2k; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "spanning or grid_kernel or c4 or tile" > $OUT/span.log 2>&1; echo "rc=$?" >> $OUT/span.log
for th in 32 64 128; do
  CLAW_GRID_TH=$th timeout 300 python bench.py --config c4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $OUT/c4_th$th.json 2>/dev/null
done
for th in 64 128 256; do
  CLAW_GRID_TH=$th timeout 300 python bench.py --config c5 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $OUT/c5_th$th.json 2>/dev/null
done
tail -n 5 $OUT/span.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('%-20s %.2f G/s  kernel %.4f ms  frac %.3f' % ('$f'.split('/')[-1], d['value']/1e9, r['avg_launch_ms'], r['frac']))"; done
