#!/bin/bash
# where do the paper workload's regrid spikes come from: phase trace of 3 bench runs
OUT=gpurun_out/r01_3k; mkdir -p $OUT
for rep in 1 2 3; do
  CLAW_TRACE_PLAN=1 timeout 300 python bench.py --config paper --steps 40 --warmup 4 --no-cpu-baseline --no-e2e > $OUT/paper_$rep.json 2>$OUT/paper_$rep.err
done
for rep in 1 2 3; do python -c "
import json; d=json.loads(open('$OUT/paper_$rep.json').read().strip().splitlines()[-1]); c=d['config']
print('paper_$rep %.3f G/s  %.4f ms/step regrid %.2f ms x %d' % (d['value']/1e9, d['ms_per_step'], c['regrid_ms_mean'], c['regrids']))"
awk '\$NF=="ms" && \$(NF-1)+0 > 4.0' $OUT/paper_$rep.err | sort | uniq -c | sort -rn | head -20; done
