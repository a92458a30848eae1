#!/bin/bash
# C2/C3 latency anatomy: kernel timeline (torch.profiler/CUPTI) + ncu launch list
OUT=gpurun_out/r01y; mkdir -p $OUT
export OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python scripts/trace_c3.py c3 > $OUT/trace_c3.json 2> $OUT/trace_c3.err
timeout 300 python scripts/trace_c3.py c2 > $OUT/trace_c2.json 2> $OUT/trace_c2.err
timeout 300 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_c3.log 2>&1
cat $OUT/trace_c3.json $OUT/trace_c2.json $OUT/bench_c3.json; tail -2 $OUT/*.err
