#!/bin/bash
# Regrid phase breakdown on the paper workload (CLAW_TRACE_PLAN=1), and a CUPTI-free timeline proxy
OUT=gpurun_out/r01_3d; mkdir -p $OUT
CLAW_TRACE_PLAN=1 timeout 600 python scripts/regrid_timing.py > $OUT/regrid.txt 2> $OUT/regrid_trace.txt
tail -5 $OUT/regrid.txt; tail -60 $OUT/regrid_trace.txt
