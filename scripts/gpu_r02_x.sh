#!/bin/bash
# evidence of the round-2 defaults: C5 launch list (bench command), ncu --set full of the C5 grid kernel and the c5vc kernel
OUT=gpurun_out/r02_x; mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_grid_kernel -s 3 -c 1 -o $OUT/ncu_grid_c5 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_grid.log 2>&1
python scripts/ncu_summary.py $OUT/ncu_grid_c5.ncu-rep $OUT/ncu_grid_c5.json 12884901888 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_vc_kernel -s 3 -c 1 -o $OUT/ncu_vc_c5 -f python bench.py --config c5vc --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_vc.log 2>&1
python scripts/ncu_summary.py $OUT/ncu_vc_c5.ncu-rep $OUT/ncu_vc_c5.json 17179869184 > /dev/null 2>&1
for k in grid vc; do python -c "import json; j=json.load(open('$OUT/ncu_${k}_c5.json'))[0]; print('$k', {k: j[k] for k in ('time_ms','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','stall_share','traffic_over_algorithmic','launch__registers_per_thread')})"; done
grep -c step_grid $OUT/launches_c5.csv
