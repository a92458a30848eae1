#!/bin/bash
OUT=gpurun_out/r01_2h; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_regrid.py tests/test_gpu_paper.py tests/test_gpu_parity.py -x -q -k "regrid or paper or update or c2 or c3" > $OUT/t.log 2>&1; echo "rc=$?" >> $OUT/t.log
timeout 600 python bench.py --config paper --steps 40 --warmup 3 --no-cpu-baseline > $OUT/paper.json 2> $OUT/paper.err
OUT=$OUT timeout 300 python scripts/trace_c3.py paper > $OUT/trace_paper.json 2>&1
OUT=$OUT timeout 300 python scripts/trace_c3.py c3 > $OUT/trace_c3.json 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:step_kernel --launch-skip 9 --launch-count 1 -o $OUT/ncu_paper_l3 python scripts/prof_hier.py --config paper --steps 3 > $OUT/ncu_paper.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:step_kernel --launch-skip 13 --launch-count 1 -o $OUT/ncu_c3_l3 python scripts/prof_hier.py --config c3 --steps 3 > $OUT/ncu_c3.log 2>&1
tail -n 3 $OUT/t.log; cat $OUT/paper.json | cut -c1-600; cat $OUT/trace_paper.json $OUT/trace_c3.json; tail -n 3 $OUT/ncu_paper.log $OUT/ncu_c3.log
