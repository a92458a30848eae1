#!/bin/bash
# generic tiles: balanced row split (default) vs 64+remainder; th cap 32
OUT=gpurun_out/r01_4r; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lane.py tests/test_gpu_side.py tests/test_gpu_paper.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for rep in 1 2 3; do
  for v in "bal" "nobal" "th32"; do
    case $v in bal) E="";; nobal) E="CLAW_GEN_BALANCE=0";; th32) E="CLAW_GEN_TH=32";; esac
    env $E timeout 300 python bench.py --config paper --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/paper_${v}_$rep.json 2>/dev/null
  done
done
for v in bal nobal; do case $v in bal) E="";; nobal) E="CLAW_GEN_BALANCE=0";; esac
  env $E timeout 300 python bench.py --config c3 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/c3_$v.json 2>/dev/null
  env $E timeout 300 python bench.py --config c2 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/c2_$v.json 2>/dev/null
done
tail -2 $OUT/pytest.log
for f in $OUT/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); c=d['config']
rg=c.get('regrid_ms_mean'); n=c.get('regrids') or 0
steps = (d['ms_per_step']*d['steps'] - (rg or 0)*n)/d['steps']
print('%-20s %.4f ms/step  steps-only %.4f  regrid %s' % ('$f'.split('/')[-1], d['ms_per_step'], steps, rg))"; done
