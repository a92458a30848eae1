#!/bin/bash
# warps per CTA: 4 (default) vs 2 vs 1 (sub-wave launches balance better with small CTAs)
OUT=gpurun_out/r01_4w; mkdir -p $OUT
for rep in 1 2; do for v in "" build/variants/libclaw_kw2.so build/variants/libclaw_kw1.so; do
  tag=$(basename "${v:-kw4}" .so | sed 's/libclaw_//')_$rep
  CLAW_LIB=$v timeout 300 python bench.py --config c3 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/c3_$tag.json 2>/dev/null
  CLAW_LIB=$v timeout 300 python bench.py --config c2 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/c2_$tag.json 2>/dev/null
  CLAW_LIB=$v timeout 300 python bench.py --config paper --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/paper_$tag.json 2>/dev/null
  CLAW_LIB=$v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_$tag.json 2>/dev/null
done; done
CLAW_LIB=build/variants/libclaw_kw1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lane.py -x -q > $OUT/pytest_kw1.log 2>&1; echo "rc=$?" >> $OUT/pytest_kw1.log
tail -2 $OUT/pytest_kw1.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); c=d['config']
rg=c.get('regrid_ms_mean'); n=c.get('regrids') or 0
steps = (d['ms_per_step']*d['steps'] - (rg or 0)*n)/d['steps']
print('%-18s %.4f ms/step  steps-only %.4f  %.2f G/s' % ('$f'.split('/')[-1], d['ms_per_step'], steps, d['value']/1e9))"; done
