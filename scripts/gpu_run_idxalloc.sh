#!/bin/bash
# Index streams (int4 staging loads) allocating in L1 (idxalloc) vs L1::no_allocate (cur); both L2 evict_first.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for t in cur idxalloc; do echo "== $t"; NUMPMP_LIB=build/variants/lib_$t.so timeout 300 python scripts/lib_bitcheck.py; NUMPMP_LIB=build/variants/lib_$t.so NUMPMP_PAIR_TILE_TAU=100 timeout 300 python scripts/lib_bitcheck.py; done > gpurun_out/idxalloc_bitcheck.txt 2>&1
for c in P C B E; do CFG=$c bash scripts/gpu_ab_libs.sh cur idxalloc; done > gpurun_out/ab_idxalloc.txt 2>&1
cat gpurun_out/idxalloc_bitcheck.txt gpurun_out/ab_idxalloc.txt
