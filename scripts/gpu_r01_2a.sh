#!/bin/bash
# session-2 state check: full gpu suite, smoke, default bench, C4 and C3 benches
OUT=gpurun_out/r01_2a; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --config c4 --steps 50 --warmup 5 --no-e2e > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 600 python bench.py --config c3 --steps 50 --warmup 5 --no-e2e > $OUT/bench_c3.json 2> $OUT/bench_c3.err
tail -3 $OUT/smoke.log $OUT/gpu_all.log
cat $OUT/bench.json $OUT/bench_c4.json $OUT/bench_c3.json
