#!/bin/bash
# branch-free march tail (halo-row sources from a prologue table) vs previous build; GPU suite
OUT=gpurun_out/r02_z; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
for i in 1 2; do
  for v in base prev; do
    lib=build/variants/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
    CLAW_LIB=$lib timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_${v}_$i.json 2> $OUT/c5_${v}_$i.err
    CLAW_LIB=$lib timeout 600 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c4_${v}_$i.json 2> $OUT/c4_${v}_$i.err
    CLAW_LIB=$lib timeout 600 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/c3_${v}_$i.json 2> $OUT/c3_${v}_$i.err
  done
done
tail -n 3 $OUT/gpu_all.log
for f in $OUT/c5_*.json $OUT/c4_*.json $OUT/c3_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'frac', round(j['roofline']['frac'],4), 'ms_per_step', round(j['ms_per_step'],4))" 2>&1 | tail -1)"; done
