#!/bin/bash
# grid kernel: 8 strips per CTA (dynamic shared ring, CLAW_GRID_KW=8) vs the default 4; rowcopy tests of both
OUT=gpurun_out/r02_cf; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_rowcopy.py tests/test_gpu_parity.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
CLAW_LIB=build/variants/libclaw_kw8.so timeout 900 python -m pytest tests/test_gpu_rowcopy.py tests/test_gpu_parity.py -q -x > $OUT/tests_kw8.log 2>&1; echo "rc=$?" >> $OUT/tests_kw8.log
tail -n 2 $OUT/tests.log $OUT/tests_kw8.log
for i in 1 2; do
  for v in base kw8; do
    lib=build/variants/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
    CLAW_LIB=$lib timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_${v}_$i.json 2> $OUT/c5_${v}_$i.err
    CLAW_LIB=$lib timeout 600 python bench.py --config c4 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c4_${v}_$i.json 2> $OUT/c4_${v}_$i.err
  done
done
for f in $OUT/*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'frac', round(j['roofline']['frac'],4))" 2>&1 | tail -1)"; done
