#!/bin/bash
# vc kernel (per-cell speed max, shuffled left kappas), bench --gpus N spawn path in TEST MODE through the stand-in NCCL
OUT=gpurun_out/r02_m; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_vc.py tests/test_gpu_multirank.py -q -x > $OUT/vc.log 2>&1; echo "rc=$?" >> $OUT/vc.log
timeout 600 python bench.py --config c5vc --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5vc.json 2> $OUT/c5vc.err
gcc -O2 -shared -fPIC -o /tmp/libncclshim.so tests/nccl_shim/ncclshim.c -ldl
for n in 2 4; do
  CLAW_NCCL_LIB=/tmp/libncclshim.so timeout 900 python bench.py --gpus $n --config c4 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/shim_c4_n$n.json 2> $OUT/shim_c4_n$n.err
  CLAW_NCCL_LIB=/tmp/libncclshim.so timeout 900 python bench.py --gpus $n --config c5vc --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/shim_c5vc_n$n.json 2> $OUT/shim_c5vc_n$n.err
done
tail -n 3 $OUT/vc.log
python -c "import json; j=json.load(open('$OUT/c5vc.json')); print('c5vc', round(j['value']/1e9,3), j['roofline']['frac'])"
for f in $OUT/shim_*.json; do echo "$f $(python -c "import json; j=json.load(open('$f')); print(j['n_gpus'], round(j['value']/1e9,3), j.get('test_mode','')[:40], [c['nccl_nranks'] for c in j['per_rank']['comm']])")"; done
grep -h "NCCL communicator" $OUT/shim_*.err | head -4
