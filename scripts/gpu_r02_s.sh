#!/bin/bash
# vc kernel with 16-byte L1 row copies, warps per CTA 4 (default) vs 1 / 2 / 3, RC 0 for reference; vc GPU tests
OUT=gpurun_out/r02_s; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_vc.py tests/test_gpu_multirank.py -q -x > $OUT/vc.log 2>&1; echo "rc=$?" >> $OUT/vc.log
for i in 1 2; do
  for v in base vckw1 vckw2 vckw3; do
    lib=build/variants/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
    CLAW_LIB=$lib timeout 600 python bench.py --config c5vc --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5vc_${v}_$i.json 2> $OUT/c5vc_${v}_$i.err
  done
done
CLAW_ROWCOPY=0 timeout 600 python bench.py --config c5vc --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5vc_rc0.json 2> $OUT/c5vc_rc0.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_vc_kernel -s 3 -c 1 -o $OUT/ncu_vc_c5 -f python bench.py --config c5vc --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_vc.log 2>&1
python scripts/ncu_summary.py $OUT/ncu_vc_c5.ncu-rep $OUT/ncu_vc_c5.json 17179869184 > /dev/null 2>&1
tail -n 3 $OUT/vc.log
for f in $OUT/c5vc_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'frac', round(j['roofline']['frac'],4), 'launch_ms', round(j['roofline']['avg_launch_ms'],4))" 2>&1 | tail -1)"; done
python -c "import json; j=json.load(open('$OUT/ncu_vc_c5.json'))[0]; print({k: j[k] for k in ('time_ms','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','stall_share','traffic_over_algorithmic','l1tex__t_sector_hit_rate.pct')})"
