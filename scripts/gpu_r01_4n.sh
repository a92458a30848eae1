#!/bin/bash
# CFL read-back wait by stream polling vs blocking sync; wide kernel on C3's sparse lattice
OUT=gpurun_out/r01_4n; mkdir -p $OUT
for rep in 1 2; do for sp in 1 0; do for cfg in c1 c2 c3; do
  CLAW_SPIN=$sp timeout 300 python bench.py --config $cfg --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/${cfg}_spin${sp}_$rep.json 2>/dev/null
done; done; done
for sp in 1 0; do CLAW_SPIN=$sp timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5_spin${sp}.json 2>/dev/null; done
CLAW_GRID_WIDE=1 timeout 300 python bench.py --config c3 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/c3_wide.json 2>/dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('%-20s %.3f G/s  %.4f ms/step' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step']))"; done
