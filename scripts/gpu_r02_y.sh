#!/bin/bash
# 8-phase fast loop (compile-time ring slots) vs 4-phase; grid / rowcopy / parity tests
OUT=gpurun_out/r02_y; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_rowcopy.py tests/test_gpu_parity.py tests/test_gpu_long.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
for i in 1 2; do
  for v in base ph4; do
    lib=build/variants/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
    CLAW_LIB=$lib timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_${v}_$i.json 2> $OUT/c5_${v}_$i.err
    CLAW_LIB=$lib timeout 600 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c4_${v}_$i.json 2> $OUT/c4_${v}_$i.err
  done
done
tail -n 3 $OUT/tests.log
for f in $OUT/c5_*.json $OUT/c4_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'frac', round(j['roofline']['frac'],4), 'launch_ms', round(j['roofline']['avg_launch_ms'],4))" 2>&1 | tail -1)"; done
