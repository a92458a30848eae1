#!/bin/bash
# HEAD check: smoke, full GPU suite, default bench line
OUT=gpurun_out/r02_cc; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
timeout 900 python bench.py > $OUT/bench_c5.json 2> $OUT/bench_c5.err
tail -n 2 $OUT/smoke.log; tail -n 3 $OUT/gpu_all.log
python -c "import json; j=json.load(open('$OUT/bench_c5.json')); print(round(j['value']/1e9,3), j['roofline']['frac'], j['ms_per_step'], j['e2e']['value'], j['clocks'])"
