#!/bin/bash
# van Leer quotient without the correctly rounded division's slow-path branch: full GPU suite; paper workload A/B vs previous build; ncu of its level-3 lane kernel
OUT=gpurun_out/r02_bq; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
tail -n 4 $OUT/gpu_all.log
for i in 1 2; do
  for v in base vldiv; do
    lib=build/variants/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
    CLAW_LIB=$lib timeout 600 python bench.py --config paper --steps 24 --warmup 8 --no-cpu-baseline --no-e2e > $OUT/paper_${v}_$i.json 2> $OUT/paper_${v}_$i.err
  done
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:step_lane_kernel -s 40 -c 1 -o $OUT/lane_paper -f python bench.py --config paper --steps 4 --warmup 9 --no-cpu-baseline --no-e2e > $OUT/ncu_lane_paper.log 2>&1
for f in $OUT/paper_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); r=j['roofline']; print(round(j['value']/1e9,3), 'ms_per_step', round(j['ms_per_step'],4), 'avg_launch_ms', round(r['avg_launch_ms'],4), 'regrid_ms', j['config'].get('regrid_ms_mean'))" 2>&1 | tail -1)"; done
