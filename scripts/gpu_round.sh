#!/bin/bash
# usage: scripts/gpu_round.sh TAG   (runs on the GPU box via gpurun)
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import torch;print(torch.cuda.get_device_name(0))" > $OUT/dev.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 python bench.py --config c4 --steps 20 --warmup 5 --no-e2e > $OUT/bench_c4.json 2> $OUT/bench_c4.err
tail -5 $OUT/pytest_gpu.log; cat $OUT/bench.json $OUT/bench_c4.json; tail -3 $OUT/bench.err
