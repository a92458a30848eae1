#!/bin/bash
# full bench line + reference arm + ncu evidence for profiles/
OUT=gpurun_out/r01k; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 900 python bench.py --config c4 > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 900 python bench.py --config c2 --steps 20 --warmup 3 > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_ -s 3 -c 1 -o $OUT/prof_c5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_c5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_ -s 3 -c 1 -o $OUT/prof_c4 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_c4.log 2>&1
cat $OUT/bench_default.json $OUT/bench_reference.json
