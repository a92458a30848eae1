#!/bin/bash
# final validation: smoke, full GPU suite, default bench line
OUT=gpurun_out/r01_4q; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo "rc=$?" >> $OUT/bench_default.err
tail -2 $OUT/smoke.log; tail -2 $OUT/gpu_all.log; cut -c1-400 $OUT/bench_default.json; tail -1 $OUT/bench_default.err
