#!/bin/bash
# device-side regrid fill + update rects + NEXT-4 paper workload
OUT=gpurun_out/r01_2e; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_regrid.py tests/test_gpu_paper.py -x -q > $OUT/regrid.log 2>&1; echo "rc=$?" >> $OUT/regrid.log
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
CLAW_TRACE_PLAN=1 timeout 900 python bench.py --config paper --steps 40 --warmup 3 > $OUT/paper.json 2> $OUT/paper.err
timeout 600 python bench.py --config c3 --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --regrid 8 > $OUT/c3_regrid8.json 2> $OUT/c3_regrid8.err
tail -n 30 $OUT/regrid.log; tail -n 3 $OUT/gpu_all.log; tail -n 40 $OUT/paper.err; cat $OUT/paper.json $OUT/c3_regrid8.json
