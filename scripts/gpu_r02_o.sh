#!/bin/bash
# RC 1 grid kernel variants: ring depth / prefetch distance, streaming stores, L2 eviction hints
OUT=gpurun_out/r02_o; mkdir -p $OUT
run() {  # name lib
  for i in 1 2; do
    CLAW_LIB=$2 timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_$1_$i.json 2> $OUT/c5_$1_$i.err
    CLAW_LIB=$2 timeout 600 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c4_$1_$i.json 2> $OUT/c4_$1_$i.err
  done
}
run base paper_1808_02638_b200/libclaw.so
for v in g16p9 g16p13 stcs hint hintstcs; do run $v build/variants/libclaw_$v.so; done
for f in $OUT/c5_*.json $OUT/c4_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'frac', round(j['roofline']['frac'],4), 'launch_ms', round(j['roofline']['avg_launch_ms'],4))" 2>&1 | tail -1)"; done
