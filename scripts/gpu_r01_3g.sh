#!/bin/bash
# lane/side tests; regrid spikes: lazy vs eager module loading; paper bench lane on/off/auto x2
OUT=gpurun_out/r01_3g; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_lane.py tests/test_gpu_side.py -x -q > $OUT/pytest_lane.log 2>&1; echo "rc=$?" >> $OUT/pytest_lane.log
timeout 600 python scripts/regrid_timing.py > $OUT/regrid_lazy.txt 2>&1
CUDA_MODULE_LOADING=EAGER timeout 600 python scripts/regrid_timing.py > $OUT/regrid_eager.txt 2>&1
for rep in 1 2; do for L in 1 0 auto; do
  if [ $L = auto ]; then unset CLAW_LANE; else export CLAW_LANE=$L; fi
  CUDA_MODULE_LOADING=EAGER timeout 300 python bench.py --config paper --steps 40 --warmup 4 --no-cpu-baseline --no-e2e > $OUT/paper_l${L}_$rep.json 2>$OUT/paper_l${L}_$rep.err
done; done
unset CLAW_LANE
tail -3 $OUT/pytest_lane.log; cat $OUT/regrid_lazy.txt $OUT/regrid_eager.txt
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); c=d['config']
print('%-18s %.3f G/s  %.4f ms/step regrid %.2f ms x %d' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], c['regrid_ms_mean'], c['regrids']))"; done
