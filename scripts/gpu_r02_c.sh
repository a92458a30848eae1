#!/bin/bash
# round 2 first box call: smoke, full GPU suite (incl. long parity), bench lines, sanitizers
OUT=gpurun_out/r02_c; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=30 > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 600 python bench.py --config c4 --steps 50 --warmup 5 > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 600 python bench.py --config c3 --steps 50 --warmup 5 > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for part in grid generic hier regrid; do
    timeout 600 $CS --tool $tool --target-processes all --print-limit 20 python scripts/sanitize.py $part > $OUT/san_${tool}_${part}.log 2>&1
    echo "rc=$?" >> $OUT/san_${tool}_${part}.log
  done
done
tail -n 3 $OUT/smoke.log $OUT/gpu_all.log | cat
cat $OUT/bench_default.json $OUT/bench_c4.json $OUT/bench_c3.json $OUT/bench_ref.json
for f in $OUT/san_*.log; do echo "$f: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|rc=' $f | tr '\n' ' ')"; done
