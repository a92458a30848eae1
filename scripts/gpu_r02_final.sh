#!/bin/bash
# round-2 final evidence: smoke, full GPU suite, bench lines of every config (default C5 with e2e and
# cpu_baseline), the reference arm, launch list of the default bench command, ncu --set full of the
# dominant kernels (C5 grid, C4 grid, c5vc vc), per-rank step times
OUT=${OUT:-gpurun_out/r02_final}; mkdir -p $OUT; export OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
timeout 900 python bench.py > $OUT/bench_c5.json 2> $OUT/bench_c5.err
for c in c4 c3 c2 c1 c5vc paper; do
  timeout 900 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_launches.log 2>&1
NCU="ncu --set full --import-source on --clock-control none"
timeout 900 $NCU -k regex:step_grid_kernel -s 2 -c 1 -o $OUT/grid_c5 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_grid_c5.log 2>&1
timeout 900 $NCU -k regex:step_grid_kernel -s 2 -c 1 -o $OUT/grid_c4 -f python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_grid_c4.log 2>&1
timeout 900 $NCU -k regex:step_vc_kernel -s 2 -c 1 -o $OUT/vc_c5vc -f python bench.py --config c5vc --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_vc.log 2>&1
timeout 600 python scripts/rank_time.py c5 20 1 2 4 8 > $OUT/rank_c5.jsonl 2> $OUT/rank_c5.err
timeout 300 python scripts/trace_batch.py c3 10 > $OUT/tb_c3.json 2> $OUT/tb_c3.err
timeout 300 python scripts/trace_batch.py c2 10 > $OUT/tb_c2.json 2> $OUT/tb_c2.err
tail -n 2 $OUT/smoke.log; tail -n 4 $OUT/gpu_all.log
for f in $OUT/bench_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); r=j.get('roofline') or {}; print(round(j['value']/1e9,4), 'frac', r.get('frac'), 'ms', round(j['ms_per_step'],4), 'e2e', (j.get('e2e') or {}).get('value'))" 2>&1 | tail -1)"; done
ls -la $OUT | head -50
