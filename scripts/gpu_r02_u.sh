#!/bin/bash
# batched hierarchy timelines (claw_advance_hierarchy_n, 10 coarse steps per sync)
OUT=gpurun_out/r02_u; mkdir -p $OUT; export OUT
for c in c2 c3; do timeout 300 python scripts/trace_batch.py $c 10 > $OUT/tb_$c.json 2> $OUT/tb_$c.err; done
cat $OUT/tb_*.json; tail -2 $OUT/tb_c2.err
