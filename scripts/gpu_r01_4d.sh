#!/bin/bash
# bench.py N>1 flow through libclaw's NCCL path with the stand-in NCCL (processes share the GPU): TEST MODE
OUT=gpurun_out/r01_4d; mkdir -p $OUT
gcc -O2 -shared -fPIC -o /tmp/libncclshim.so tests/nccl_shim/ncclshim.c -ldl
for n in 2 4; do
  CLAW_NCCL_LIB=/tmp/libncclshim.so timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 5 --warmup 3 --config c4 --no-cpu-baseline > $OUT/bench_shim_n$n.json 2> $OUT/bench_shim_n$n.err; echo "rc=$?" >> $OUT/bench_shim_n$n.err
done
for n in 2 4; do cut -c1-260 $OUT/bench_shim_n$n.json; python -c "
import json; d=json.loads(open('$OUT/bench_shim_n$n.json').read().strip().splitlines()[-1]); print(d.get('test_mode'), d['config']['parallelism'], d['gpu_launches'], d['e2e']['value'])"; tail -1 $OUT/bench_shim_n$n.err; done
