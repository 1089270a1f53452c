#!/bin/bash
# Row-mode link pass: rounds of 512 staged through registers (base) vs cp.async rounds of 512 / 1024.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for t in base row1024; do echo "== $t"; NUMPMP_LIB=build/variants/lib_$t.so timeout 300 python scripts/lib_bitcheck.py; done > gpurun_out/row_bitcheck.txt 2>&1
for c in C B; do CFG=$c bash scripts/gpu_ab_libs.sh base row512a row1024; done > gpurun_out/ab_row.txt 2>&1
cat gpurun_out/row_bitcheck.txt gpurun_out/ab_row.txt
