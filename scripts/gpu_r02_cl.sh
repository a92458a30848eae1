#!/bin/bash
# grid tile heights re-swept on the round's final kernel (CLAW_GRID_TH forced vs the makespan choice)
OUT=gpurun_out/r02_cl; mkdir -p $OUT
run() { # cfg th tag
  if [ "$2" = auto ]; then env -u CLAW_GRID_TH timeout 300 python bench.py --config $1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/$1_$3.json 2> $OUT/$1_$3.err
  else CLAW_GRID_TH=$2 timeout 300 python bench.py --config $1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/$1_$3.json 2> $OUT/$1_$3.err; fi
  python -c "import json; j=json.loads(open('$OUT/$1_$3.json').read().strip().splitlines()[-1]); r=j['roofline']; print('$1 $3', round(j['value']/1e9,2), 'G frac', round(r['frac'],4), 'launch_ms', round(r['avg_launch_ms'],4))"
}
for c in c4 c5; do run $c auto auto1; done
for th in 32 64 96 128 160 192 224 256 320 384; do run c4 $th th$th; done
for th in 64 128 192 256 320 384 448 512; do run c5 $th th$th; done
for c in c4 c5; do run $c auto auto2; done
