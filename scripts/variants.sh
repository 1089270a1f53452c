#!/bin/bash
# Build tuning variants of libnumpmp_cuda.so into build/variants/ (here, on
# CPU), then run them on the GPU box with scripts/sweep.sh.
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
build() {  # name, extra nvcc flags...
  local name=$1; shift
  nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -shared \
    -Iinclude "$@" -o build/variants/lib_$name.so \
    paper_2509_10722_b200/csrc/pmp_solver.cu paper_2509_10722_b200/csrc/host_gen.cpp -ldl -cudart static &
}
build base
build stage256 -DNUMPMP_STAGE_INTS=256
build stage1024 -DNUMPMP_STAGE_INTS=1024
build unroll8 -DNUMPMP_GATHER_UNROLL=8
build unroll2 -DNUMPMP_GATHER_UNROLL=2
build minb3 -DNUMPMP_MIN_BLOCKS=3
build minb5 -DNUMPMP_MIN_BLOCKS=5
build warps4 -DNUMPMP_WARPS=4 -DNUMPMP_MIN_BLOCKS=8
wait
ls -la build/variants
