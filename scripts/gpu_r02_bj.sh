#!/bin/bash
# timelines of C3 / C2 / C1 after the latency-bound kernel changes; ncu of C3's level-3 grid kernel and level-1 lane kernel
OUT=gpurun_out/r02_bj; mkdir -p $OUT; export OUT
timeout 300 python scripts/trace_batch.py c3 10 > $OUT/tb_c3.json 2> $OUT/tb_c3.err
timeout 300 python scripts/trace_batch.py c2 10 > $OUT/tb_c2.json 2> $OUT/tb_c2.err
NCU="ncu --set full --import-source on --clock-control none"
timeout 600 $NCU -k regex:step_grid_kernel -s 24 -c 1 -o $OUT/c3l3 -f python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_c3l3.log 2>&1
timeout 600 $NCU -k regex:step_lane_kernel -s 9 -c 1 -o $OUT/c3lane -f python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_c3lane.log 2>&1
cat $OUT/tb_c3.json $OUT/tb_c2.json
