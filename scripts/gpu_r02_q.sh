#!/bin/bash
# RC 1 with L1-allocating 16-byte copies: warps per CTA (neighbouring strips share an SM's L1), 16-slot ring
OUT=gpurun_out/r02_q; mkdir -p $OUT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,l1tex__t_sector_hit_rate.pct
V="ca16 ca16kw2 ca16kw4 ca16g16p9"
for v in $V; do
  CLAW_LIB=build/variants/libclaw_$v.so timeout 600 ncu --metrics $M --clock-control none -k regex:step_grid_kernel -s 3 -c 1 --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/m_$v.csv 2> $OUT/m_$v.err
done
for i in 1 2; do
  for v in base $V; do
    lib=build/variants/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
    CLAW_LIB=$lib timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_${v}_$i.json 2> $OUT/c5_${v}_$i.err
    CLAW_LIB=$lib timeout 600 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c4_${v}_$i.json 2> $OUT/c4_${v}_$i.err
  done
done
for f in $OUT/m_*.csv; do echo "== $f"; grep -E "dram__|lts__|gpu__time|l1tex" $f | awk -F'","' '{print $(NF-3), $(NF-2), $(NF-1), $NF}'; done
for f in $OUT/c5_*.json $OUT/c4_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'frac', round(j['roofline']['frac'],4), 'launch_ms', round(j['roofline']['avg_launch_ms'],4))" 2>&1 | tail -1)"; done
