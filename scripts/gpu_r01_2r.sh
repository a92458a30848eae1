#!/bin/bash
# multi-rank skeleton on one GPU (TEST MODE --exchange host), reference arm under torchrun, default bench
OUT=gpurun_out/r01_2r; mkdir -p $OUT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --exchange host --config c4 --no-cpu-baseline > $OUT/mr2.json 2> $OUT/mr2.err; echo "rc=$?" >> $OUT/mr2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > $OUT/ref2.json 2> $OUT/ref2.err; echo "rc=$?" >> $OUT/ref2.err
/usr/bin/time -v timeout 900 python bench.py > $OUT/default.json 2> $OUT/default.err; echo "rc=$?" >> $OUT/default.err
cat $OUT/mr2.json | cut -c1-400; tail -n 2 $OUT/mr2.err; cat $OUT/ref2.json | cut -c1-300; tail -n 1 $OUT/ref2.err
python -c "
import json; d=json.loads(open('$OUT/default.json').read().strip().splitlines()[-1]); print(d['value']/1e9, d['roofline']['frac'], d['cpu_baseline'])"
grep "Elapsed" $OUT/default.err
