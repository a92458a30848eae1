#!/bin/bash
# wave-aware grid tile heights (C4 192, C5 384 rows): GPU suite, bench lines, sweep; vc occupancy variant; launch list
OUT=gpurun_out/r02_j; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_auto.json 2> $OUT/c5_auto.err
timeout 600 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c4_auto.json 2> $OUT/c4_auto.err
for th in 128 192 256 320; do
  CLAW_GRID_TH=$th timeout 600 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c4_th$th.json 2> $OUT/c4_th$th.err
done
for th in 256 384 512; do
  CLAW_GRID_TH=$th timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_th$th.json 2> $OUT/c5_th$th.err
done
CLAW_LIB=build/variants/libclaw_vc16.so timeout 600 python bench.py --config c5vc --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5vc_vc16.json 2> $OUT/c5vc_vc16.err
timeout 600 python bench.py --config c5vc --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5vc_base.json 2> $OUT/c5vc_base.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/launches.log 2>&1
tail -n 3 $OUT/gpu_all.log
for f in $OUT/*.json; do echo "$f $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'frac', round(j['roofline']['frac'],4), 'launch_ms', round(j['roofline']['avg_launch_ms'],4))")"; done
