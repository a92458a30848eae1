#!/bin/bash
# regridding inside the timed region (NEXT-3 measurement)
OUT=gpurun_out/r01_2c; mkdir -p $OUT
for cfg in c2 c3; do
  for k in 0 4 1; do
    timeout 600 python bench.py --config $cfg --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --regrid $k > $OUT/${cfg}_regrid$k.json 2> $OUT/${cfg}_regrid$k.err
  done
done
timeout 600 python bench.py --config c3 --steps 40 --warmup 5 --regrid 4 > $OUT/c3_regrid4_full.json 2> $OUT/c3_regrid4_full.err
for f in $OUT/*.json; do echo $f; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); c=d['config']
print(' ms/step %.3f  G/s %.2f regrids %s regrid_ms %s patches %s' % (d['ms_per_step'], d['value']/1e9, c.get('regrids'), c.get('regrid_ms_mean'), c.get('patches_after')))"; done
tail -n 3 $OUT/*.err
