#!/bin/bash
OUT=gpurun_out/r01_2m; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
for cfg in c3 paper; do
  timeout 600 python bench.py --config $cfg --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/$cfg.json 2> $OUT/$cfg.err
done
timeout 600 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --path 1 > $OUT/c5_generic.json 2> $OUT/c5_generic.err
OUT=$OUT timeout 300 python scripts/trace_c3.py c3 > $OUT/trace_c3.json 2>&1
tail -n 3 $OUT/gpu_all.log
for f in $OUT/c3.json $OUT/paper.json $OUT/c5_generic.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('%-20s %.3f G/s  %.4f ms/step  kernel %.4f ms frac %.3f' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], r['avg_launch_ms'], r['frac']))"; done
cat $OUT/trace_c3.json | tail -n 1
