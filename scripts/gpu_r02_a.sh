#!/bin/bash
# round 2 baseline: smoke, full GPU suite, default bench line
OUT=gpurun_out/r02_a; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --durations=30 > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 600 python bench.py --config c4 --steps 50 --warmup 5 > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 600 python bench.py --config c3 --steps 50 --warmup 5 > $OUT/bench_c3.json 2> $OUT/bench_c3.err
tail -n 3 $OUT/smoke.log $OUT/gpu_all.log | cat
cat $OUT/bench_default.json $OUT/bench_c4.json $OUT/bench_c3.json
