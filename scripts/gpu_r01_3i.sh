#!/bin/bash
# grid kernel without the halo-row pointer registers: full GPU suite + C5/C4 (x2)
OUT=gpurun_out/r01_3i; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_all.log 2>&1; echo "rc=$?" >> $OUT/pytest_all.log
for rep in 1 2; do
  timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_$rep.json 2>$OUT/c5_$rep.err
  timeout 300 python bench.py --config c4 --steps 80 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c4_$rep.json 2>$OUT/c4_$rep.err
done
tail -3 $OUT/pytest_all.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('%-12s %.2f G/s  %.4f ms/step frac %.4f' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], r['frac']))"; done
