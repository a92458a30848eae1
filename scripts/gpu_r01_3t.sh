#!/bin/bash
# bench.py multi-rank skeleton (torchrun) on one GPU via --exchange host (test mode)
OUT=gpurun_out/r01_3t; mkdir -p $OUT
timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --config c4 --exchange host > $OUT/bench_n2.json 2> $OUT/bench_n2.err; echo "rc=$?" >> $OUT/bench_n2.err
timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 5 --warmup 3 --config c4 --exchange host --path 1 --no-e2e > $OUT/bench_n4.json 2> $OUT/bench_n4.err; echo "rc=$?" >> $OUT/bench_n4.err
timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 3 --warmup 1 --impl reference > $OUT/bench_ref_n2.json 2> $OUT/bench_ref_n2.err; echo "rc=$?" >> $OUT/bench_ref_n2.err
cat $OUT/bench_n2.json $OUT/bench_n4.json $OUT/bench_ref_n2.json; tail -3 $OUT/*.err
timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_n1_torchrun.json 2> $OUT/bench_n1_torchrun.err; echo "rc=$?" >> $OUT/bench_n1_torchrun.err
cat $OUT/bench_n1_torchrun.json | cut -c1-300; tail -2 $OUT/bench_n1_torchrun.err
