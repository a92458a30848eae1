#!/bin/bash
# Build tuning variants of libclaw.so into build/variants/ (same sources, -D knobs)
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
for v in "$@"; do
  IFS=_ read -r minb grd <<< "$v"
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
    -Xcompiler -fPIC -shared -DCLAW_MINB=$minb -DCLAW_GRD=$grd -I include \
    -o build/variants/libclaw_${v}.so paper_1808_02638_b200/csrc/claw_kernels.cu \
    paper_1808_02638_b200/csrc/claw_host.cpp -ldl &
done
wait
ls build/variants
