#!/bin/bash
OUT=gpurun_out/r01_4e; mkdir -p $OUT
CLAW_TRACE_PLAN=1 timeout 300 python bench.py --config paper --steps 40 --warmup 4 --no-cpu-baseline --no-e2e > $OUT/paper.json 2>$OUT/paper.err
CLAW_TRACE_PLAN=1 timeout 300 python scripts/regrid_timing.py > $OUT/rt.txt 2>$OUT/rt.err
for f in $OUT/paper.err $OUT/rt.err; do echo "== $f"; grep -E "\] (sat|d2h|BR|nest-split|flag) " $f | awk '{k=$1" "$2" "$3; a[k]+=$4; n[k]++; if ($4>m[k]) m[k]=$4} END {for (k in a) printf "%-22s mean %6.2f max %6.2f n=%d\n", k, a[k]/n[k], m[k], n[k]}' | sort; done
