#!/bin/bash
# Row-mode link pass gather batch 8 (default) / 12 / 16, C and P.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for t in rowu8 rowu16; do echo "== $t"; NUMPMP_LIB=build/variants/lib_$t.so timeout 300 python scripts/lib_bitcheck.py; done > gpurun_out/rowu_bitcheck.txt 2>&1
for c in C P; do CFG=$c bash scripts/gpu_ab_libs.sh rowu8 rowu12 rowu16; done > gpurun_out/ab_rowu.txt 2>&1
cat gpurun_out/rowu_bitcheck.txt gpurun_out/ab_rowu.txt
