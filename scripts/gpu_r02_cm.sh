#!/bin/bash
# makespan tile heights capped at 192 rows: full GPU suite + bench lines (c5vc against the old 384)
OUT=gpurun_out/r02_cm; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log; tail -n 2 $OUT/gpu_all.log
run() { # cfg th tag
  if [ "$2" = auto ]; then timeout 300 python bench.py --config $1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/$1_$3.json 2> $OUT/$1_$3.err
  else CLAW_GRID_TH=$2 timeout 300 python bench.py --config $1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/$1_$3.json 2> $OUT/$1_$3.err; fi
  python -c "import json; j=json.loads(open('$OUT/$1_$3.json').read().strip().splitlines()[-1]); r=j['roofline']; print('$1 $3', round(j['value']/1e9,2), 'G frac', round(r['frac'],4), 'ms', round(j['ms_per_step'],4))"
}
for i in 1 2; do
  run c5 auto auto$i; run c5 384 th384_$i; run c4 auto auto$i
  run c5vc auto auto$i; run c5vc 384 th384_$i; run c5vc 256 th256_$i
  run paper auto auto$i; run c3 auto auto$i
done
