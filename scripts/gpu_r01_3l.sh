#!/bin/bash
# geometric pool growth; glibc malloc env (no mmap/trim churn) vs default on the paper workload
OUT=gpurun_out/r01_3l; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_regrid.py tests/test_gpu_paper.py tests/test_gpu_parity.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for rep in 1 2 3; do
  CLAW_TRACE_PLAN=1 timeout 300 python bench.py --config paper --steps 40 --warmup 4 --no-cpu-baseline --no-e2e > $OUT/paper_$rep.json 2>$OUT/paper_$rep.err
  CLAW_TRACE_PLAN=1 MALLOC_MMAP_THRESHOLD_=33554432 MALLOC_TRIM_THRESHOLD_=4294967296 MALLOC_TOP_PAD_=268435456 timeout 300 python bench.py --config paper --steps 40 --warmup 4 --no-cpu-baseline --no-e2e > $OUT/paperm_$rep.json 2>$OUT/paperm_$rep.err
done
tail -2 $OUT/pytest.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); c=d['config']
print('%-14s %.3f G/s  %.4f ms/step regrid %.2f ms x %d' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], c['regrid_ms_mean'], c['regrids']))"; done
for f in $OUT/*.err; do echo "$f: $(grep -c . $f) lines; max phases:"; grep -E "\] (plan|alloc|cluster|kernels) " $f | sort -k5 -n -r | head -4; done
