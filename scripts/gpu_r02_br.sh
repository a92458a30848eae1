#!/bin/bash
# halo-lane kernel: ghost-cell rectangle map (one load per segment resolution instead of the rectangle search) vs previous build
OUT=gpurun_out/r02_br; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_lane.py tests/test_gpu_paper.py tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_side.py tests/test_gpu_reflux.py tests/test_gpu_regrid.py tests/test_gpu_long.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
tail -n 3 $OUT/tests.log
for i in 1 2; do
  for v in base vl; do
    lib=build/variants/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
    CLAW_LIB=$lib timeout 600 python bench.py --config paper --steps 24 --warmup 8 --no-cpu-baseline --no-e2e > $OUT/paper_${v}_$i.json 2> $OUT/paper_${v}_$i.err
    for c in c3 c2; do CLAW_LIB=$lib timeout 600 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/${c}_${v}_$i.json 2> $OUT/${c}_${v}_$i.err; done
  done
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:step_lane_kernel -s 40 -c 1 -o $OUT/lane_paper -f python bench.py --config paper --steps 4 --warmup 9 --no-cpu-baseline --no-e2e > $OUT/ncu_lane_paper.log 2>&1
for f in $OUT/*_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); r=j['roofline']; print(round(j['value']/1e9,3), 'ms_per_step', round(j['ms_per_step'],4), 'avg_launch_ms', round(r['avg_launch_ms'],4))" 2>&1 | tail -1)"; done
