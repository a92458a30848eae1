#!/bin/bash
OUT=gpurun_out/r01_2g; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_regrid.py tests/test_gpu_paper.py -x -q > $OUT/regrid.log 2>&1; echo "rc=$?" >> $OUT/regrid.log
CLAW_TRACE_PLAN=1 timeout 900 python bench.py --config paper --steps 40 --warmup 3 --no-cpu-baseline > $OUT/paper.json 2> $OUT/paper.err
OUT=$OUT timeout 300 python scripts/trace_c3.py paper > $OUT/trace_paper.json 2>&1
tail -n 3 $OUT/regrid.log; grep -v "^\[plan" $OUT/paper.err | tail -n 24; cat $OUT/paper.json; cat $OUT/trace_paper.json
python - <<'PY'
import collections
rows=[l for l in open("gpurun_out/r01_2g/trace_paper.txt")]
agg=collections.defaultdict(lambda:[0,0.0])
gap=0.0
for l in rows:
    p=l.split()
    d=float(p[2]); g=float(p[4]); nm=" ".join(p[5:])[:60]
    agg[nm][0]+=1; agg[nm][1]+=d; gap+=g
for k,v in sorted(agg.items(), key=lambda kv:-kv[1][1]): print("%6d %10.1f us  %s"%(v[0],v[1],k))
print("total gaps us", gap)
PY
