#!/bin/bash
OUT=gpurun_out/r01_2j; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_graph.py -x -q > $OUT/graph.log 2>&1; echo "rc=$?" >> $OUT/graph.log
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
for cfg in c2 c3 paper; do
  timeout 600 python bench.py --config $cfg --steps 40 --warmup 5 --no-cpu-baseline > $OUT/$cfg.json 2> $OUT/$cfg.err
  CLAW_NO_GRAPH=1 timeout 600 python bench.py --config $cfg --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${cfg}_nograph.json 2> $OUT/${cfg}_nograph.err
done
OUT=$OUT timeout 300 python scripts/trace_c3.py c3 > $OUT/trace_c3.json 2>&1
tail -n 30 $OUT/graph.log; tail -n 3 $OUT/gpu_all.log
for f in $OUT/c2.json $OUT/c2_nograph.json $OUT/c3.json $OUT/c3_nograph.json $OUT/paper.json $OUT/paper_nograph.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('%-28s %.3f G/s  %.4f ms/step  kernel share %.2f e2e %s' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], r['kernel_share_of_step'] or 0, (d.get('e2e') or {}).get('value')))"; done
cat $OUT/trace_c3.json; tail -n 5 $OUT/c3.err
