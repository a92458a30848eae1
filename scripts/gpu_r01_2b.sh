#!/bin/bash
# regridding on the GPU + pool; full gpu suite
OUT=gpurun_out/r01_2b; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_regrid.py -x -q > $OUT/regrid.log 2>&1; echo "rc=$?" >> $OUT/regrid.log
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
tail -n 30 $OUT/regrid.log; tail -n 5 $OUT/gpu_all.log
