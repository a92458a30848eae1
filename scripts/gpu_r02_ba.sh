#!/bin/bash
# session-4 re-entry baseline: smoke, full GPU suite, default bench line, c5vc line
OUT=gpurun_out/r02_ba; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 1800 python -m pytest tests -m gpu -q --durations=25 > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 600 python bench.py --config c5vc --steps 30 --warmup 5 --no-cpu-baseline > $OUT/bench_c5vc.json 2> $OUT/bench_c5vc.err
tail -n 3 $OUT/smoke.log; tail -n 40 $OUT/gpu_all.log
for f in $OUT/bench_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'frac', round(j['roofline']['frac'],4), 'ms', round(j['ms_per_step'],4))" 2>&1 | tail -1)"; done
