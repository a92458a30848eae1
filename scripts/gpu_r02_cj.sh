#!/bin/bash
# band split: interior tile heights any multiple of 4 (makespan over near-integral waves) vs multiples of my
OUT=gpurun_out/r02_cj; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_nccl_path.py tests/test_gpu_parity.py tests/test_gpu_rowcopy.py tests/test_gpu_vc.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
tail -n 3 $OUT/tests.log
for v in base; do
  lib=build/variants/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
  for i in 1 2; do
    CLAW_LIB=$lib timeout 600 python scripts/rank_time.py c5 20 1 2 4 8 > $OUT/rank_c5_${v}_$i.jsonl 2> $OUT/rank_c5_${v}_$i.err
  done
  CLAW_LIB=$lib timeout 600 python scripts/rank_time.py c5vc 20 1 4 8 > $OUT/rank_c5vc_${v}.jsonl 2> $OUT/rank_c5vc_${v}.err
done
for f in $OUT/rank_*.jsonl; do echo "== $f"; python -c "
import json
for l in open('$f'):
    j=json.loads(l); print(j['N'], j['rank'], round(j['ms_per_step'],4), j['projected_speedup'] and round(j['projected_speedup'],3))
"; done
