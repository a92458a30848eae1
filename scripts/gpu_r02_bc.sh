#!/bin/bash
# band split (thin edge launch): multirank / NCCL-path tests; per-rank step time of C5 / c5vc at N = 1, 2, 4, 8 (new vs previous build)
OUT=gpurun_out/r02_bc; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_nccl_path.py tests/test_gpu_parity.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
tail -n 3 $OUT/tests.log
for v in new prev; do
  lib=build/variants/libclaw_$v.so; [ $v = new ] && lib=paper_1808_02638_b200/libclaw.so
  CLAW_LIB=$lib timeout 600 python scripts/rank_time.py c5 20 1 2 4 8 > $OUT/rank_c5_$v.jsonl 2> $OUT/rank_c5_$v.err
  CLAW_LIB=$lib timeout 600 python scripts/rank_time.py c5vc 20 1 2 4 8 > $OUT/rank_c5vc_$v.jsonl 2> $OUT/rank_c5vc_$v.err
done
for f in $OUT/rank_*.jsonl; do echo "== $f"; python -c "
import json,sys
for l in open('$f'):
    j=json.loads(l); print(j['N'], j['rank'], round(j['ms_per_step'],4), round(j['step_kernel_ms_per_step'],4), j['launches_per_step'], j['projected_speedup'] and round(j['projected_speedup'],2))
"; tail -2 ${f%.jsonl}.err; done
