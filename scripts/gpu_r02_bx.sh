#!/bin/bash
# interpolation specs not zero-filled before the planner writes them: regrid phases, paper line, regrid + paper GPU tests
OUT=gpurun_out/r02_bx; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_regrid.py tests/test_gpu_paper.py tests/test_gpu_parity.py tests/test_gpu_long.py tests/test_gpu_lane.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
tail -n 2 $OUT/tests.log
CLAW_TRACE_PLAN=1 timeout 600 python scripts/regrid_timing.py > $OUT/regrid_timing.txt 2> $OUT/trace_plan.txt
tail -n 3 $OUT/regrid_timing.txt; tail -n 38 $OUT/trace_plan.txt
for i in 1 2; do timeout 600 python bench.py --config paper --steps 24 --warmup 8 --no-cpu-baseline --no-e2e > $OUT/paper_$i.json 2> $OUT/paper_$i.err; done
for f in $OUT/*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); r=j['roofline']; print(round(j['value']/1e9,3), 'ms_per_step', round(j['ms_per_step'],4), 'avg_launch_ms', round(r['avg_launch_ms'],4), 'regrid_ms', j['config'].get('regrid_ms_mean'))" 2>&1 | tail -1)"; done
