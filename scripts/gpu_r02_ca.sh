#!/bin/bash
# bench.py --gpus 2 on multi-level configs through libclaw's NCCL path with the test stand-in NCCL (TEST MODE: processes share one GPU)
OUT=gpurun_out/r02_ca; mkdir -p $OUT
gcc -O2 -shared -fPIC -o $OUT/libncclshim.so tests/nccl_shim/ncclshim.c -ldl
for c in c2 c3; do
  CLAW_NCCL_LIB=$OUT/libncclshim.so timeout 900 python bench.py --config $c --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_${c}_n2.json 2> $OUT/bench_${c}_n2.err; echo "rc=$?" >> $OUT/bench_${c}_n2.err
done
cat $OUT/bench_*_n2.json; tail -5 $OUT/bench_c3_n2.err
