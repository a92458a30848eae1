#!/bin/bash
# grid-kernel row copies: RC 1 (16-byte per-lane cp.async) and RC 2 (cp.async.bulk) vs RC 0;
# GPU suite under RC 1 (default) and RC 2; C5 / C4 lines per RC; ncu of RC 1 and RC 2
OUT=gpurun_out/r02_n; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/gpu_rc1.log 2>&1; echo "rc=$?" >> $OUT/gpu_rc1.log
CLAW_ROWCOPY=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_long.py tests/test_gpu_multirank.py -m gpu -q -x > $OUT/gpu_rc2.log 2>&1; echo "rc=$?" >> $OUT/gpu_rc2.log
for rc in 0 1 2; do
  CLAW_ROWCOPY=$rc timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_rc$rc.json 2> $OUT/c5_rc$rc.err
  CLAW_ROWCOPY=$rc timeout 600 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c4_rc$rc.json 2> $OUT/c4_rc$rc.err
done
for rc in 1 2; do
  CLAW_ROWCOPY=$rc timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_grid_kernel -s 3 -c 1 -o $OUT/ncu_grid_c5_rc$rc -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_rc$rc.log 2>&1
  python scripts/ncu_summary.py $OUT/ncu_grid_c5_rc$rc.ncu-rep $OUT/ncu_grid_c5_rc$rc.json 12884901888 > /dev/null 2>&1
done
tail -n 3 $OUT/gpu_rc1.log $OUT/gpu_rc2.log
for f in $OUT/c5_rc*.json $OUT/c4_rc*.json; do echo "$f $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'frac', round(j['roofline']['frac'],4), 'launch_ms', round(j['roofline']['avg_launch_ms'],4))")"; done
for rc in 1 2; do python -c "import json; j=json.load(open('$OUT/ncu_grid_c5_rc$rc.json'))[0]; print($rc, {k: j[k] for k in ('time_ms','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','stall_share','traffic_over_algorithmic')})"; done
