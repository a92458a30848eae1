#!/bin/bash
# vc kernel tile heights by its own resident-warp count (12) vs the grid kernel's (16)
# (measured and dropped: profiles/r02_vc_makespan.txt; the CLAW_VC_MAKESPAN knob and abvar/ variant are gone)
OUT=gpurun_out/r02_ck; mkdir -p $OUT; ls -la abvar build/variants > $OUT/ls.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_vc.py tests/test_gpu_rowcopy.py tests/test_gpu_multirank.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
tail -n 3 $OUT/tests.log
for i in 1 2; do
  for v in base novcms; do
    lib=abvar/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
    CLAW_LIB=$lib timeout 300 python bench.py --config c5vc --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5vc_${v}_$i.json 2> $OUT/c5vc_${v}_$i.err
    python -c "import json; j=json.loads(open('$OUT/c5vc_${v}_$i.json').read().strip().splitlines()[-1]); print('$v $i', j['value'], j['ms_per_step'], j['roofline']['frac'])"
  done
  for v in base novcms; do
    lib=abvar/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
    CLAW_LIB=$lib timeout 600 python scripts/rank_time.py c5vc 20 4 8 > $OUT/rank_c5vc_${v}_$i.jsonl 2> $OUT/rank_c5vc_${v}_$i.err
  done
done
for f in $OUT/rank_*.jsonl; do echo "== $f"; python -c "
import json
for l in open('$f'):
    j=json.loads(l); print(j['N'], j['rank'], round(j['ms_per_step'],4))
"; done
