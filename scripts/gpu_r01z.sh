#!/bin/bash
# conservation fix on the GPU + full gpu suite + C3 tile-rows sweep
OUT=gpurun_out/r01z; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_reflux.py -x -q > $OUT/reflux.log 2>&1; echo "rc=$?" >> $OUT/reflux.log
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
for tr in 16 32 64; do
  timeout 300 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --tile-rows $tr > $OUT/c3_tr$tr.json 2>&1
done
tail -5 $OUT/reflux.log $OUT/gpu_all.log
for f in $OUT/c3_tr*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['value']/1e9)"; done
