#!/bin/bash
# K1 with streaming (L1::no_allocate, L2 evict_first) loads of col_ptr / w / kind, end offset by shuffle (k1na) vs cur.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for t in cur k1na; do echo "== $t"; NUMPMP_LIB=build/variants/lib_$t.so timeout 300 python scripts/lib_bitcheck.py; NUMPMP_LIB=build/variants/lib_$t.so NUMPMP_PAIR_TILE_TAU=100 timeout 300 python scripts/lib_bitcheck.py; done > gpurun_out/k1na_bitcheck.txt 2>&1
for c in C P B E; do CFG=$c bash scripts/gpu_ab_libs.sh cur k1na; done > gpurun_out/ab_k1na.txt 2>&1
cat gpurun_out/k1na_bitcheck.txt gpurun_out/ab_k1na.txt
