#!/bin/bash
OUT=gpurun_out/r01f; mkdir -p $OUT
for v in 4_1 5_2 4_3; do
  for c in c5 c4; do
    CLAW_LIB=build/variants/libclaw_$v.so timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_${v}_$c.json 2>>$OUT/bench_err.log
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_ -s 2 -c 1 -o $OUT/prof_c5 python scripts/prof_step.py --config c5 --steps 3 > $OUT/ncu_c5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_ -s 2 -c 1 -o $OUT/prof_c4 python scripts/prof_step.py --config c4 --steps 3 > $OUT/ncu_c4.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_c5.csv python bench.py --config c5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
for f in $OUT/bench_*.json; do echo $f; python -c "import json,sys; j=json.load(open('$f')); print(j['value']/1e9, j['roofline']['frac'], j['ms_per_step'])"; done
