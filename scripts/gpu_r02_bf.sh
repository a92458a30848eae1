#!/bin/bash
# vc kernel resident warps per SM: 12 (168 registers, default) vs 14 vs 16 (128 registers, 4-byte spill)
OUT=gpurun_out/r02_bf; mkdir -p $OUT
for i in 1 2; do
  for v in base vc14 vc16; do
    lib=build/variants/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
    CLAW_LIB=$lib timeout 600 python bench.py --config c5vc --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5vc_${v}_$i.json 2> $OUT/c5vc_${v}_$i.err
  done
done
for f in $OUT/c5vc_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'frac', round(j['roofline']['frac'],4), 'ms', round(j['ms_per_step'],4))" 2>&1 | tail -1)"; done
