#!/bin/bash
# regrid phase timings of the paper workload (CLAW_TRACE_PLAN=1) and per-call wall clock
OUT=gpurun_out/r02_bv; mkdir -p $OUT
CLAW_TRACE_PLAN=1 timeout 600 python scripts/regrid_timing.py > $OUT/regrid_timing.txt 2> $OUT/trace_plan.txt
tail -8 $OUT/regrid_timing.txt; grep -c . $OUT/trace_plan.txt; tail -60 $OUT/trace_plan.txt
