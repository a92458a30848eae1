#!/bin/bash
# final validation + evidence (one warp per CTA): smoke, full GPU suite, every bench line, launch list, ncu C5/C4
OUT=gpurun_out/r01_4x; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for cfg in c4 c3 c2 c1; do timeout 600 python bench.py --config $cfg --steps 50 --warmup 5 > $OUT/bench_$cfg.json 2> $OUT/bench_$cfg.err; done
for r in 1 2 3; do timeout 600 python bench.py --config paper --steps 50 --warmup 5 > $OUT/bench_paper_$r.json 2> $OUT/bench_paper_$r.err; done
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 5 -c 40 --csv --log-file $OUT/launches_c5.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_grid -s 2 -c 1 -o $OUT/ncu_c5 python scripts/prof_step.py --config c5 --steps 3 > $OUT/ncu_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_grid -s 2 -c 1 -o $OUT/ncu_c4 python scripts/prof_step.py --config c4 --steps 3 > $OUT/ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_grid -s 20 -c 1 -o $OUT/ncu_c3_l3 python scripts/prof_hier.py --config c3 --steps 3 > $OUT/ncu_c3.log 2>&1
tail -n 2 $OUT/smoke.log $OUT/gpu_all.log | cat
for f in $OUT/bench_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('%-24s %.3f G/s  ms/step %.4f frac %s e2e %s' % ('$f'.split('/')[-1], d['value']/1e9, d['ms_per_step'], r.get('frac'), (d.get('e2e') or {}).get('value')))"; done
