#!/bin/bash
# vc kernel: copy issued after the row's warp barrier (racecheck), tests, c5vc line
OUT=gpurun_out/r02_ac; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck synccheck memcheck; do timeout 600 $CS --tool $tool --target-processes all --print-limit 20 python scripts/sanitize.py vc > $OUT/san_${tool}_vc.log 2>&1; echo "rc=$?" >> $OUT/san_${tool}_vc.log; done
timeout 900 python -m pytest tests/test_gpu_vc.py tests/test_gpu_rowcopy.py tests/test_gpu_multirank.py -q -x > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
for i in 1 2; do timeout 600 python bench.py --config c5vc --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c5vc_$i.json 2> $OUT/c5vc_$i.err; done
for f in $OUT/san_*.log; do echo "$f: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|rc=' $f | tr '\n' ' ')"; done
tail -n 2 $OUT/tests.log
for f in $OUT/c5vc_*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); print(round(j['value']/1e9,3), 'frac', round(j['roofline']['frac'],4))" 2>&1 | tail -1)"; done
