#!/bin/bash
# ncu (source level) of the paper workload's level-3 halo-lane kernel; the workload's launch list
OUT=gpurun_out/r02_bp; mkdir -p $OUT
NCU="ncu --set full --import-source on --clock-control none"
timeout 900 $NCU -k regex:step_lane_kernel -s 40 -c 3 -o $OUT/lane_paper -f python bench.py --config paper --steps 4 --warmup 9 --no-cpu-baseline --no-e2e > $OUT/ncu_lane_paper.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none -c 200 --csv --log-file $OUT/launches_paper.csv python bench.py --config paper --steps 4 --warmup 9 --no-cpu-baseline --no-e2e > $OUT/ncu_launches.log 2>&1
ls -la $OUT
