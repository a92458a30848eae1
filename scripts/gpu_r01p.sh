#!/bin/bash
OUT=gpurun_out/r01p; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_ -s 3 -c 1 -o $OUT/prof_gen_c5 python bench.py --path 1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_gen_c5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_ -s 8 -c 3 -o $OUT/prof_c3 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_c3.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_launch_c3.log 2>&1
echo done
