#!/bin/bash
# planner refactor check + regrid phase trace
OUT=gpurun_out/r01_2d; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
CLAW_TRACE_PLAN=1 timeout 600 python bench.py --config c3 --steps 16 --warmup 3 --no-e2e --no-cpu-baseline --regrid 4 > $OUT/c3_regrid4.json 2> $OUT/c3_regrid4.err
tail -n 3 $OUT/gpu_all.log; tail -n 60 $OUT/c3_regrid4.err; cat $OUT/c3_regrid4.json
