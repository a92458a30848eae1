#!/bin/bash
OUT=gpurun_out/r01_3n; mkdir -p $OUT
for rep in 1 2; do
  CLAW_TRACE_PLAN=1 timeout 300 python bench.py --config paper --steps 40 --warmup 4 --no-cpu-baseline --no-e2e > $OUT/paper_$rep.json 2>$OUT/paper_$rep.err
done
for f in $OUT/*.err; do echo "== $f"; grep -E "\] [a-z+-]+ +[0-9.]+ ms" $f | awk '{k=$1" "$2" "$3; a[k]+=$4; n[k]++; if ($4>m[k]) m[k]=$4} END {for (k in a) printf "%-24s mean %6.2f max %6.2f n=%d\n", k, a[k]/n[k], m[k], n[k]}' | sort | grep -v "plan L1"; done
