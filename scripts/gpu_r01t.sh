#!/bin/bash
# round-1 evidence: default bench line, per-config lines, reference arm, ncu
# summaries (small files only: gpurun brings back <= 64 MiB)
OUT=gpurun_out/r01t; mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 900 python bench.py --config c4 > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 900 python bench.py --config c3 --steps 10 --warmup 3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 900 python bench.py --config c2 --steps 20 --warmup 3 > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 900 python bench.py --config c1 --steps 20 --warmup 3 > $OUT/bench_c1.json 2> $OUT/bench_c1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
for c in c5 c4 gen_c5; do
  args="--config ${c#gen_}"; [ "$c" = gen_c5 ] && args="--config c5 --path 1"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_ -s 3 -c 1 -o /tmp/prof_$c python bench.py $args --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_$c.log 2>&1
  alg=12884901888; [ "$c" = c4 ] && alg=3221225472
  python scripts/ncu_summary.py /tmp/prof_$c.ncu-rep $OUT/ncu_summary_$c.json $alg > /dev/null 2>&1
  ncu -i /tmp/prof_$c.ncu-rep --page details --csv > $OUT/ncu_details_$c.csv 2>/dev/null
done
cp /tmp/prof_c5.ncu-rep $OUT/prof_c5.ncu-rep
du -sh $OUT
