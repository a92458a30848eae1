#!/bin/bash
# refresh of the secondary bench lines after the interpolation slices
OUT=gpurun_out/r01_4u; mkdir -p $OUT
for cfg in c3 c2 c1; do
  timeout 600 python bench.py --config $cfg --steps 50 --warmup 5 > $OUT/bench_$cfg.json 2> $OUT/bench_$cfg.err
done
for r in 1 2 3; do timeout 600 python bench.py --config paper --steps 50 --warmup 5 > $OUT/bench_paper_$r.json 2> $OUT/bench_paper_$r.err; done
for f in $OUT/bench_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('%-24s %.3f G/s  ms/step %.4f e2e %s cpu %s' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value')))"; done
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 600 python bench.py --config c4 --steps 50 --warmup 5 > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for f in $OUT/bench_default.json $OUT/bench_c4.json $OUT/bench_reference.json; do cut -c1-200 $f; done
