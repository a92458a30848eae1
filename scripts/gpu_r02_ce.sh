#!/bin/bash
# grid kernel: 2 strips per CTA (CLAW_GRID_KW=2) vs the default 4
OUT=gpurun_out/r02_ce; mkdir -p $OUT
for i in 1 2; do
  for v in base kw2; do
    lib=build/variants/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
    CLAW_LIB=$lib timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_${v}_$i.json 2> $OUT/c5_${v}_$i.err
    CLAW_LIB=$lib timeout 600 python bench.py --config c4 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c4_${v}_$i.json 2> $OUT/c4_${v}_$i.err
  done
done
for f in $OUT/*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'frac', round(j['roofline']['frac'],4))" 2>&1 | tail -1)"; done
