#!/bin/bash
# makespan cap 192 for the MC limiter (van Leer and vc levels uncapped): GPU suite + bench lines
OUT=gpurun_out/r02_co; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log; tail -n 2 $OUT/gpu_all.log
for c in c5 c4 c5vc paper c3; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/$c.json 2> $OUT/$c.err
  python -c "import json; j=json.loads(open('$OUT/$c.json').read().strip().splitlines()[-1]); r=j['roofline']; print('$c', round(j['value']/1e9,3), 'G frac', round(r['frac'],4), 'ms', round(j['ms_per_step'],4))"
done
timeout 600 python bench.py > $OUT/bench_c5_default.json 2> $OUT/bench_c5_default.err; tail -c 400 $OUT/bench_c5_default.json
