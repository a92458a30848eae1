#!/bin/bash
# update_rect_kernel<R>: 16-byte child-pair loads vs previous build; updating tests
OUT=gpurun_out/r02_cd; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_long.py tests/test_gpu_parity.py tests/test_gpu_multirank_hier.py tests/test_gpu_reflux.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
tail -n 2 $OUT/tests.log
for i in 1 2; do
  for v in base dist; do
    lib=build/variants/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
    for c in c3 c2; do CLAW_LIB=$lib timeout 600 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/${c}_${v}_$i.json 2> $OUT/${c}_${v}_$i.err; done
  done
done
OUT=$OUT timeout 300 python scripts/trace_batch.py c3 10 > $OUT/tb_c3.json 2> $OUT/tb_c3.err; grep update_rect $OUT/trace_batch_c3.txt | head -4
for f in $OUT/c*_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'ms_per_step', round(j['ms_per_step'],4))" 2>&1 | tail -1)"; done
