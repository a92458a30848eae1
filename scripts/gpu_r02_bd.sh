#!/bin/bash
# band-split tests; vc kernel cubic reciprocal (RCP3) vs two Newton steps: accuracy probe, vc tests, c5vc lines
OUT=gpurun_out/r02_bd; mkdir -p $OUT
./scripts/rcp_check > $OUT/rcp_check.json 2>&1
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_nccl_path.py tests/test_gpu_vc.py tests/test_gpu_parity.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
for i in 1 2; do
  for v in base rcp2; do
    lib=build/variants/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
    CLAW_LIB=$lib timeout 600 python bench.py --config c5vc --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5vc_${v}_$i.json 2> $OUT/c5vc_${v}_$i.err
  done
done
cat $OUT/rcp_check.json; tail -n 3 $OUT/tests.log
for f in $OUT/c5vc_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'frac', round(j['roofline']['frac'],4), 'ms', round(j['ms_per_step'],4))" 2>&1 | tail -1)"; done
