#!/bin/bash
# lane kernel: tile records carry their patch's off / mx / my and patches their region rectangles (first segment after one load latency) vs previous build; tile-rows 4 vs auto on C1 / C2
OUT=gpurun_out/r02_bl; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_lane.py tests/test_gpu_parity.py tests/test_gpu_paper.py tests/test_gpu_multirank.py tests/test_gpu_nccl_path.py tests/test_gpu_side.py tests/test_gpu_reflux.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
for i in 1 2; do
  for v in base lat1; do
    lib=build/variants/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
    for c in c3 c2 c1; do CLAW_LIB=$lib timeout 600 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/${c}_${v}_$i.json 2> $OUT/${c}_${v}_$i.err; done
    CLAW_LIB=$lib timeout 600 python bench.py --config paper --steps 24 --warmup 8 --no-cpu-baseline --no-e2e > $OUT/paper_${v}_$i.json 2> $OUT/paper_${v}_$i.err
  done
  for c in c2 c1; do timeout 600 python bench.py --config $c --tile-rows 4 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/${c}_th4_$i.json 2> $OUT/${c}_th4_$i.err; done
done
tail -n 2 $OUT/tests.log
for f in $OUT/*_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'ms_per_step', round(j['ms_per_step'],4))" 2>&1 | tail -1)"; done
