#!/bin/bash
# Multi-route stream tiles with the next tile's offsets loaded one tile ahead (qpf) vs base, on E.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for t in base qpf; do echo "== $t"; NUMPMP_LIB=build/variants/lib_$t.so NUMPMP_PAIR_TILE_TAU=100 timeout 300 python scripts/lib_bitcheck.py; done > gpurun_out/qpf_bitcheck.txt 2>&1
CFG=E bash scripts/gpu_ab_libs.sh base qpf > gpurun_out/ab_qpf.txt 2>&1
cat gpurun_out/qpf_bitcheck.txt gpurun_out/ab_qpf.txt
