#!/bin/bash
OUT=gpurun_out/r01_2s; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_side.py -x -q > $OUT/side.log 2>&1; echo "rc=$?" >> $OUT/side.log
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
for sd in 0 1; do
  for cfg in c3 paper; do
    CLAW_SIDE=$sd timeout 600 python bench.py --config $cfg --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${cfg}_side$sd.json 2> $OUT/${cfg}_side$sd.err
  done
  CLAW_SIDE=$sd timeout 600 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --path 1 > $OUT/c5gen_side$sd.json 2> $OUT/c5gen_side$sd.err
done
tail -n 5 $OUT/side.log; tail -n 3 $OUT/gpu_all.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('%-22s %.3f G/s  %.4f ms/step  kernel %.4f ms  frac %.3f' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], r['avg_launch_ms'], r['frac']))"; done
