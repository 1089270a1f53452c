#!/bin/bash
# Flat gathers (NUMPMP_FLAT_GATHER=1 build) vs base: bit-identity, then interleaved benches C/B/E/D.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for t in base flat; do echo "== $t"; NUMPMP_LIB=build/variants/lib_$t.so timeout 300 python scripts/lib_bitcheck.py; done > gpurun_out/flat_bitcheck.txt 2>&1
cat gpurun_out/flat_bitcheck.txt
for c in C B E; do CFG=$c bash scripts/gpu_ab_libs.sh base flat; done > gpurun_out/ab_flat.txt 2>&1
cat gpurun_out/ab_flat.txt
