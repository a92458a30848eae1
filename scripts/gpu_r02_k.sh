#!/bin/bash
# neighbour preload: GPU suite + C5/C4 lines + ncu; reference arm of c5vc
OUT=gpurun_out/r02_k; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
timeout 600 python bench.py --steps 50 --warmup 5 > $OUT/c5.json 2> $OUT/c5.err
timeout 600 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu-baseline > $OUT/c4.json 2> $OUT/c4.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_grid_kernel -s 3 -c 1 -o $OUT/ncu_grid_c5 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_grid.log 2>&1
python scripts/ncu_summary.py $OUT/ncu_grid_c5.ncu-rep $OUT/ncu_grid_c5.json 12884901888 > /dev/null 2>&1
timeout 900 python bench.py --config c5vc --impl reference --steps 3 --warmup 1 > $OUT/ref_c5vc.json 2> $OUT/ref_c5vc.err
tail -n 3 $OUT/gpu_all.log
for f in $OUT/c5.json $OUT/c4.json; do echo "$f $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'frac', round(j['roofline']['frac'],4), 'launch_ms', round(j['roofline']['avg_launch_ms'],4))")"; done
python -c "import json; j=json.load(open('$OUT/ncu_grid_c5.json'))[0]; print({k: j[k] for k in ('time_ms','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','stall_share','traffic_over_algorithmic')})"
cat $OUT/ref_c5vc.json
