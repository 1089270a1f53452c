#!/bin/bash
# Row-mode link pass reading row_ptr with L1::no_allocate + evict_first (rpna) vs cur.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for t in cur rpna; do echo "== $t"; NUMPMP_LIB=build/variants/lib_$t.so timeout 300 python scripts/lib_bitcheck.py; NUMPMP_LIB=build/variants/lib_$t.so NUMPMP_PAIR_TILE_TAU=100 timeout 300 python scripts/lib_bitcheck.py; done > gpurun_out/rpna_bitcheck.txt 2>&1
for c in P C; do CFG=$c bash scripts/gpu_ab_libs.sh cur rpna; done > gpurun_out/ab_rpna.txt 2>&1
cat gpurun_out/rpna_bitcheck.txt gpurun_out/ab_rpna.txt
