#!/bin/bash
OUT=gpurun_out/r02_l; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_vc.py tests/test_gpu_multirank.py tests/test_gpu_nccl_path.py -q -x > $OUT/vc_mr.log 2>&1; echo "rc=$?" >> $OUT/vc_mr.log
timeout 600 python bench.py --config c5vc --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5vc.json 2> $OUT/c5vc.err
tail -n 5 $OUT/vc_mr.log
python -c "import json; j=json.load(open('$OUT/c5vc.json')); print(round(j['value']/1e9,3), j['roofline']['frac'])"
