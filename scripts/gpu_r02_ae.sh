#!/bin/bash
# C3: sparse-lattice tile height 32 (auto) / 16 / 8
OUT=gpurun_out/r02_ae; mkdir -p $OUT; export OUT
for i in 1 2; do
  for th in 0 16 8; do
    if [ $th = 0 ]; then unset CLAW_SPARSE_TH; else export CLAW_SPARSE_TH=$th; fi
    timeout 600 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/c3_th${th}_$i.json 2> $OUT/c3_th${th}_$i.err
  done
done
unset CLAW_SPARSE_TH
CLAW_SPARSE_TH=16 timeout 300 python scripts/trace_batch.py c3 10 > $OUT/tb_c3_th16.json 2>&1; mv $OUT/trace_batch_c3.txt $OUT/trace_batch_c3_th16.txt
for f in $OUT/c3_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'ms_per_step', round(j['ms_per_step'],4))" 2>&1 | tail -1)"; done
