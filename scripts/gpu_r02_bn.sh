#!/bin/bash
# grid kernel: empty-issue tail block (the tile's last 4 rows prefetch nothing) vs previous build; grid tests
OUT=gpurun_out/r02_bn; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rowcopy.py tests/test_gpu_multirank.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
for i in 1 2; do
  for v in base fin; do
    lib=build/variants/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
    for c in c3 c2 c1; do CLAW_LIB=$lib timeout 600 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/${c}_${v}_$i.json 2> $OUT/${c}_${v}_$i.err; done
    CLAW_LIB=$lib timeout 600 python bench.py --config c4 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c4_${v}_$i.json 2> $OUT/c4_${v}_$i.err
    CLAW_LIB=$lib timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_${v}_$i.json 2> $OUT/c5_${v}_$i.err
  done
done
tail -n 2 $OUT/tests.log
for f in $OUT/*_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'ms_per_step', round(j['ms_per_step'],4))" 2>&1 | tail -1)"; done
