#!/bin/bash
# makespan cap 192 (vc levels keep the uncapped rule) vs the uncapped build (abvar/libclaw_cap512.so, -DCLAW_SPAN_AUTO_MAX=512)
OUT=gpurun_out/r02_cn; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_vc.py tests/test_gpu_rowcopy.py tests/test_gpu_parity.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log; tail -n 2 $OUT/tests.log
for i in 1 2; do
  for v in new cap512; do
    lib=abvar/libclaw_$v.so; [ $v = new ] && lib=paper_1808_02638_b200/libclaw.so
    for c in c5 c5vc c3 paper c2; do
      CLAW_LIB=$lib timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/${c}_${v}_$i.json 2> $OUT/${c}_${v}_$i.err
      python -c "import json; j=json.loads(open('$OUT/${c}_${v}_$i.json').read().strip().splitlines()[-1]); r=j['roofline']; print('$c $v $i', round(j['value']/1e9,3), 'G frac', round(r['frac'],4), 'ms', round(j['ms_per_step'],4))"
    done
  done
done
