#!/bin/bash
# vc parity + bench line, re-run sanitizers on the fixed lane kernel / initcheck paths
OUT=gpurun_out/r02_d; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_vc.py -q -x --durations=10 > $OUT/vc.log 2>&1; echo "rc=$?" >> $OUT/vc.log
timeout 600 python bench.py --config c5vc --steps 30 --warmup 5 --no-cpu-baseline > $OUT/bench_c5vc.json 2> $OUT/bench_c5vc.err
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck initcheck; do
  for part in generic regrid grid; do
    timeout 600 $CS --tool $tool --target-processes all --print-limit 20 python scripts/sanitize.py $part > $OUT/san_${tool}_${part}.log 2>&1
    echo "rc=$?" >> $OUT/san_${tool}_${part}.log
  done
done
python - > $OUT/vc_small.log 2>&1 <<'PY'
import numpy as np, oracle
from paper_1808_02638_b200 import binding, workloads as W
d = W.uniform_level(2, 2, 16, 16); aux = W.random_media(d, 1); q0 = W.random_ic(d, 1)
g = binding.Claw(W.DOMAIN, W.EXTRAP, 4, 2, device=0); g.set_level(1, d, q0); g.set_aux(1, aux)
o = oracle.Oracle(W.DOMAIN, W.EXTRAP, 4, 2); o.set_level(1, d, q0); o.set_aux(1, aux)
dt = 0.8 * float(d["dx"][0]) / W.max_sound_speed(aux, d)
for n in range(3):
    g.fill_ghost(1, 0); o.fill_ghost(1, 0)
    print("cfl", g.advance_level(1, dt), o.advance_level(1, dt))
    a, b = g.read_level(1), o.read_level(1)
    print("step", n, "err", np.abs(a - b).max(), "argmax", np.unravel_index(np.abs(a-b).argmax(), (4, 3, 16, 16)))
PY
tail -n 3 $OUT/vc.log; cat $OUT/vc_small.log | tail -8; cat $OUT/bench_c5vc.json; tail -3 $OUT/bench_c5vc.err
for f in $OUT/san_*.log; do echo "$f: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|rc=' $f | tr '\n' ' ')"; done
