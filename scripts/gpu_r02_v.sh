#!/bin/bash
# RC 0 vs RC 1 bitwise tests; bench lines of every config (hierarchies now timed without per-launch events)
OUT=gpurun_out/r02_v; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_rowcopy.py -q -x > $OUT/rowcopy.log 2>&1; echo "rc=$?" >> $OUT/rowcopy.log
timeout 900 python bench.py --steps 50 --warmup 5 > $OUT/c5.json 2> $OUT/c5.err
timeout 600 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu-baseline > $OUT/c4.json 2> $OUT/c4.err
timeout 600 python bench.py --config c5vc --steps 30 --warmup 5 --no-cpu-baseline > $OUT/c5vc.json 2> $OUT/c5vc.err
for c in c3 c2 c1; do timeout 600 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline > $OUT/$c.json 2> $OUT/$c.err; done
timeout 900 python bench.py --config paper --steps 24 --warmup 8 --no-cpu-baseline > $OUT/paper.json 2> $OUT/paper.err
tail -n 3 $OUT/rowcopy.log
for c in c5 c4 c5vc c3 c2 c1 paper; do python -c "import json; j=json.load(open('$OUT/$c.json')); r=j['roofline']; print('$c', round(j['value']/1e9,3), 'G', round(j['ms_per_step'],4), 'ms/step', 'frac', r['frac'] and round(r['frac'],4), 'e2e', j['e2e'] and round(j['e2e']['value']/1e9,3), 'cpu', j.get('cpu_baseline') and j['cpu_baseline'].get('value'))" 2>&1 | tail -1; done
