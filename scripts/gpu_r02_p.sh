#!/bin/bash
# DRAM re-reads of the RC 1 grid kernel: L2 / DRAM sector counts for RC 0, RC 1 (.cg), RC 1 (.ca), 16-slot ring
OUT=gpurun_out/r02_p; mkdir -p $OUT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_write_lookup_miss.sum
prof() {  # name env...
  env "${@:2}" timeout 600 ncu --metrics $M --clock-control none -k regex:step_grid_kernel -s 3 -c 1 --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/m_$1.csv 2> $OUT/m_$1.err
}
prof rc0 CLAW_ROWCOPY=0
prof rc1 CLAW_ROWCOPY=1
prof ca16 CLAW_LIB=build/variants/libclaw_ca16.so
prof g16p13 CLAW_LIB=build/variants/libclaw_g16p13.so
for i in 1 2; do
  for v in base ca16 g16p13 g16p9; do
    lib=build/variants/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
    CLAW_LIB=$lib timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_${v}_$i.json 2> $OUT/c5_${v}_$i.err
  done
done
for f in $OUT/m_*.csv; do echo "== $f"; grep -E "dram__|lts__|gpu__time" $f | awk -F'","' '{print $(NF-3), $(NF-2), $(NF-1), $NF}'; done
for f in $OUT/c5_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'frac', round(j['roofline']['frac'],4), 'launch_ms', round(j['roofline']['avg_launch_ms'],4))" 2>&1 | tail -1)"; done
