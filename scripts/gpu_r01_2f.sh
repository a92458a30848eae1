#!/bin/bash
OUT=gpurun_out/r01_2f; mkdir -p $OUT
CLAW_TRACE_PLAN=1 timeout 900 python bench.py --config paper --steps 40 --warmup 3 > $OUT/paper.json 2> $OUT/paper.err
grep -v "^\[plan" $OUT/paper.err | tail -n 60; cat $OUT/paper.json
