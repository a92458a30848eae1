#!/bin/bash
# multi-rank hierarchies (claw_config.dist_level): virtual-rank and NCCL-path tests, plus the suites the change touches
OUT=gpurun_out/r02_by; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_multirank_hier.py tests/test_gpu_nccl_path.py -q -x > $OUT/tests_new.log 2>&1; echo "rc=$?" >> $OUT/tests_new.log
tail -n 40 $OUT/tests_new.log
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
tail -n 4 $OUT/gpu_all.log
