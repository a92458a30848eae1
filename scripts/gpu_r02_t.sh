#!/bin/bash
# C3 / C2 timelines with the current kernels; ncu of a C3 level-3 launch (sparse-lattice grid kernel) and a level-2 lane-kernel launch
OUT=gpurun_out/r02_t; mkdir -p $OUT
export OUT
timeout 300 python scripts/trace_c3.py c3 > $OUT/trace_c3.json 2> $OUT/trace_c3.err
timeout 300 python scripts/trace_c3.py c2 > $OUT/trace_c2.json 2> $OUT/trace_c2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_grid_kernel -s 12 -c 1 -o $OUT/ncu_c3_l3 -f python scripts/prof_hier.py --config c3 --steps 3 > $OUT/ncu_c3_l3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_lane_kernel -s 4 -c 1 -o $OUT/ncu_c3_lane -f python scripts/prof_hier.py --config c3 --steps 3 > $OUT/ncu_c3_lane.log 2>&1
for c in c3 c2; do timeout 600 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/$c.json 2> $OUT/$c.err; done
cat $OUT/trace_c3.json $OUT/trace_c2.json
for f in $OUT/c3.json $OUT/c2.json; do python -c "import json; j=json.load(open('$f')); print('$f', round(j['value']/1e9,3), j['ms_per_step'])"; done
