#!/bin/bash
# long parity runs + full GPU suite after the cleanup; compute-sanitizer on every kernel family
OUT=gpurun_out/r02_b; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_long.py -q --durations=20 > $OUT/long.log 2>&1; echo "rc=$?" >> $OUT/long.log
timeout 900 python -m pytest tests -m gpu -q -x --ignore=tests/test_gpu_long.py > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for part in grid generic hier regrid; do
    timeout 600 $CS --tool $tool --target-processes all --print-limit 20 python scripts/sanitize.py $part > $OUT/san_${tool}_${part}.log 2>&1
    echo "rc=$?" >> $OUT/san_${tool}_${part}.log
  done
done
tail -n 4 $OUT/long.log $OUT/gpu_all.log | cat
for f in $OUT/san_*.log; do echo "$f: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|rc=' $f | tr '\n' ' ')"; done
