#!/bin/bash
# vc kernel branch-free tail vs previous build; vc / rowcopy tests; C3 batched timeline
OUT=gpurun_out/r02_aa; mkdir -p $OUT; export OUT
timeout 900 python -m pytest tests/test_gpu_vc.py tests/test_gpu_rowcopy.py tests/test_gpu_multirank.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
for i in 1 2; do
  for v in base prev; do
    lib=build/variants/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
    CLAW_LIB=$lib timeout 600 python bench.py --config c5vc --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5vc_${v}_$i.json 2> $OUT/c5vc_${v}_$i.err
  done
done
timeout 300 python scripts/trace_batch.py c3 10 > $OUT/tb_c3.json 2> $OUT/tb_c3.err
tail -n 3 $OUT/tests.log
for f in $OUT/c5vc_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'frac', round(j['roofline']['frac'],4), 'ms_per_step', round(j['ms_per_step'],4))" 2>&1 | tail -1)"; done
cat $OUT/tb_c3.json
