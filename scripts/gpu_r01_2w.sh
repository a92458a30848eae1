#!/bin/bash
OUT=gpurun_out/r01_2w; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sparse" > $OUT/sparse.log 2>&1; echo "rc=$?" >> $OUT/sparse.log
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
for sp in 1 0; do
  CLAW_SPARSE=$sp timeout 600 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/c3_sparse$sp.json 2>/dev/null
done
OUT=$OUT timeout 300 python scripts/trace_c3.py c3 > $OUT/trace_c3.json 2>&1
tail -n 15 $OUT/sparse.log; tail -n 3 $OUT/gpu_all.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('%-24s %.3f G/s  %.4f ms/step' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step']))" 2>/dev/null; done
tail -n 1 $OUT/trace_c3.json
