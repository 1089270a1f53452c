#!/bin/bash
# Stream pass with the tile prologue prefetched by cp.async (NUMPMP_K1_PF=1) vs base: bit-identity, parity, A/B on C/E/B.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in 0 1; do echo "== NUMPMP_K1_PF=$v"; NUMPMP_K1_PF=$v timeout 300 python scripts/lib_bitcheck.py; NUMPMP_K1_PF=$v NUMPMP_PAIR_TILE_TAU=100 timeout 300 python scripts/lib_bitcheck.py; done > gpurun_out/pf_bitcheck.txt 2>&1
cat gpurun_out/pf_bitcheck.txt
NUMPMP_K1_PF=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "solve_matches or tiles or blocks or p2p_exchange_ranks" > gpurun_out/pytest_pf.log 2>&1; tail -2 gpurun_out/pytest_pf.log
VARIANTS="NUMPMP_K1_PF=0 NUMPMP_K1_PF=1" CFGS="C E B" bash scripts/gpu_ab_env.sh pf
