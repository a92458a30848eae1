#!/bin/bash
OUT=gpurun_out/r01_2u; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
for pdl in 1 0; do
  for cfg in c2 c3; do
    CLAW_PDL=$pdl timeout 600 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/${cfg}_pdl$pdl.json 2> $OUT/${cfg}_pdl$pdl.err
  done
  CLAW_PDL=$pdl timeout 600 python bench.py --config paper --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --regrid 0 > $OUT/paper_noregrid_pdl$pdl.json 2> $OUT/paper_pdl$pdl.err
done
OUT=$OUT timeout 300 python scripts/trace_c3.py c3 > $OUT/trace_c3.json 2>&1
tail -n 3 $OUT/gpu_all.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('%-28s %.3f G/s  %.4f ms/step' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step']))" 2>/dev/null; done
tail -n 1 $OUT/trace_c3.json
