#!/bin/bash
# single-level batched steps (K per host sync) and hierarchy-wide CFL all-reduce: NCCL-path tests, bench lines
OUT=gpurun_out/r02_bb; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_nccl_path.py tests/test_gpu_long.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
for b in 1 10; do
  timeout 600 python bench.py --batch $b --no-cpu-baseline > $OUT/c5_b$b.json 2> $OUT/c5_b$b.err
  timeout 600 python bench.py --config c4 --batch $b --steps 50 --warmup 5 --no-cpu-baseline > $OUT/c4_b$b.json 2> $OUT/c4_b$b.err
  timeout 600 python bench.py --config c1 --batch $b --steps 200 --warmup 10 --no-cpu-baseline > $OUT/c1_b$b.json 2> $OUT/c1_b$b.err
done
tail -n 3 $OUT/tests.log
for f in $OUT/c*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'frac', j['roofline']['frac'], 'ms', round(j['ms_per_step'],4), 'e2e', round(j['e2e']['value']/1e9,2))" 2>&1 | tail -1)"; done
