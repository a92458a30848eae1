#!/bin/bash
# cell_src through the ghost-cell rectangle map (flagging, side passes, reflux): full GPU suite; paper / C2 / C3 lines
OUT=gpurun_out/r02_bu; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/gpu_all.log 2>&1; echo "rc=$?" >> $OUT/gpu_all.log
tail -n 3 $OUT/gpu_all.log
for i in 1 2; do
  timeout 600 python bench.py --config paper --steps 24 --warmup 8 --no-cpu-baseline --no-e2e > $OUT/paper_$i.json 2> $OUT/paper_$i.err
done
for c in c2 c3; do timeout 600 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/${c}.json 2> $OUT/${c}.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/launches_paper.csv python bench.py --config paper --steps 4 --warmup 9 --no-cpu-baseline --no-e2e > $OUT/ncu_launches.log 2>&1
for f in $OUT/*.json; do echo "$(basename $f .json) $(python -c "import json; j=json.load(open('$f')); r=j['roofline']; print(round(j['value']/1e9,3), 'ms_per_step', round(j['ms_per_step'],4), 'avg_launch_ms', round(r['avg_launch_ms'],4), 'regrid_ms', j['config'].get('regrid_ms_mean'))" 2>&1 | tail -1)"; done
