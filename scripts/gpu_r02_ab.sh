#!/bin/bash
# compute-sanitizer on every kernel family after the round-2 row copies / branch-free tails
OUT=gpurun_out/r02_ab; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck memcheck synccheck initcheck; do
  for part in grid vc hier generic regrid; do
    timeout 600 $CS --tool $tool --target-processes all --print-limit 20 python scripts/sanitize.py $part > $OUT/san_${tool}_${part}.log 2>&1
    echo "rc=$?" >> $OUT/san_${tool}_${part}.log
  done
done
for f in $OUT/san_*.log; do echo "$f: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|rc=' $f | tr '\n' ' ')"; done
