#!/bin/bash
# round-2 final ncu --set full captures of the dominant kernels (one launch each, after 2 warm-up launches)
OUT=gpurun_out/r02_final; mkdir -p $OUT
NCU="ncu --set full --import-source on --clock-control none"
timeout 900 $NCU -k regex:step_grid_kernel -s 2 -c 1 -o $OUT/grid_c5 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_grid_c5.log 2>&1
timeout 900 $NCU -k regex:step_grid_kernel -s 2 -c 1 -o $OUT/grid_c4 -f python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_grid_c4.log 2>&1
timeout 900 $NCU -k regex:step_vc_kernel -s 2 -c 1 -o $OUT/vc_c5vc -f python bench.py --config c5vc --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_vc.log 2>&1
ls -la $OUT/*.ncu-rep; tail -2 $OUT/ncu_grid_c5.log
