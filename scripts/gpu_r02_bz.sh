#!/bin/bash
# per-rank coarse-step time of multi-rank hierarchies (dist_level = finest), one rank at a time on one GPU
OUT=gpurun_out/r02_bz; mkdir -p $OUT
timeout 600 python scripts/rank_time.py c3 20 1 2 4 8 > $OUT/rank_c3.jsonl 2> $OUT/rank_c3.err
timeout 600 python scripts/rank_time.py c2 20 1 2 4 > $OUT/rank_c2.jsonl 2> $OUT/rank_c2.err
cat $OUT/rank_c3.jsonl $OUT/rank_c2.jsonl; tail -3 $OUT/rank_c3.err
