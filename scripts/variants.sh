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
    paper_2509_10722_b200/csrc/pmp_solver.cu paper_2509_10722_b200/csrc/host_gen.cpp paper_2509_10722_b200/csrc/host_io.cpp -ldl -cudart static &
}
build base
build unroll4 -DNUMPMP_GATHER_UNROLL=4
build unroll12 -DNUMPMP_GATHER_UNROLL=12
wait
ls -la build/variants
