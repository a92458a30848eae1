#!/bin/bash
# full GPU suite (vc, boundary), sanitizers, vc ncu capture, vc + c5 bench
OUT=gpurun_out/r02_e; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck memcheck synccheck initcheck; do
  for part in generic regrid grid hier vc; do
    timeout 600 $CS --tool $tool --target-processes all --print-limit 20 python scripts/sanitize.py $part > $OUT/san_${tool}_${part}.log 2>&1
    echo "rc=$?" >> $OUT/san_${tool}_${part}.log
  done
done
timeout 600 python bench.py --config c5vc --steps 30 --warmup 5 --no-cpu-baseline > $OUT/bench_c5vc.json 2> $OUT/bench_c5vc.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_vc_kernel -s 2 -c 1 -o $OUT/ncu_vc_c5 -f python bench.py --config c5vc --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_vc.log 2>&1
python scripts/ncu_summary.py $OUT/ncu_vc_c5.ncu-rep $OUT/ncu_vc_c5.json 17179869184 > /dev/null 2>&1
tail -n 4 $OUT/gpu_all.log
for f in $OUT/san_*.log; do echo "$f: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|rc=' $f | tr '\n' ' ')"; done
cat $OUT/bench_c5vc.json; head -c 1500 $OUT/ncu_vc_c5.json
