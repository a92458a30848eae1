#!/bin/bash
# ghost-cell rectangle map built in parallel on the host: paper workload A/B vs the van Leer build (and C2, C1)
OUT=gpurun_out/r02_bs; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_lane.py tests/test_gpu_paper.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
tail -n 2 $OUT/tests.log
for i in 1 2 3; do
  for v in base vl; do
    lib=build/variants/libclaw_$v.so; [ $v = base ] && lib=paper_1808_02638_b200/libclaw.so
    CLAW_LIB=$lib timeout 600 python bench.py --config paper --steps 24 --warmup 8 --no-cpu-baseline --no-e2e > $OUT/paper_${v}_$i.json 2> $OUT/paper_${v}_$i.err
  done
done
for c in c2 c1; do timeout 600 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/${c}_base.json 2> $OUT/${c}_base.err; done
for f in $OUT/*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); r=j['roofline']; print(round(j['value']/1e9,3), 'ms_per_step', round(j['ms_per_step'],4), 'avg_launch_ms', round(r['avg_launch_ms'],4), 'regrid_ms', j['config'].get('regrid_ms_mean'))" 2>&1 | tail -1)"; done
