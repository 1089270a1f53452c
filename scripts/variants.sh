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
build u4_minb6 -DNUMPMP_GATHER_UNROLL=4 -DNUMPMP_MIN_BLOCKS=6
build u4_minb8 -DNUMPMP_GATHER_UNROLL=4 -DNUMPMP_MIN_BLOCKS=8
build u2_minb8 -DNUMPMP_GATHER_UNROLL=2 -DNUMPMP_MIN_BLOCKS=8
build u8_minb5 -DNUMPMP_GATHER_UNROLL=8 -DNUMPMP_MIN_BLOCKS=5
build w4_u4_minb12 -DNUMPMP_WARPS=4 -DNUMPMP_GATHER_UNROLL=4 -DNUMPMP_MIN_BLOCKS=12
wait
ls -la build/variants
