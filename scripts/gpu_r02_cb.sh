#!/bin/bash
# re-sweep after the prologue / map changes: sparse-lattice tile rows (C3 level 3) and the smallest automatic tile height
OUT=gpurun_out/r02_cb; mkdir -p $OUT
for i in 1 2; do
  for th in 32 16; do CLAW_SPARSE_TH=$th timeout 600 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/c3_sth${th}_$i.json 2> $OUT/c3_sth${th}_$i.err; done
  for m in 4 8; do
    for c in c2 c3; do CLAW_MIN_TH=$m timeout 600 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/${c}_m${m}_$i.json 2> $OUT/${c}_m${m}_$i.err; done
  done
done
for f in $OUT/*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'ms_per_step', round(j['ms_per_step'],4))" 2>&1 | tail -1)"; done
