#!/bin/bash
# Multi-route stream tiles staged in rounds of 256 (stageq) vs 512 (base): E, plus bit-identity and a pair-tile parity test.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for t in base stageq; do echo "== $t"; NUMPMP_LIB=build/variants/lib_$t.so NUMPMP_PAIR_TILE_TAU=100 timeout 300 python scripts/lib_bitcheck.py; done > gpurun_out/stageq_bitcheck.txt 2>&1
NUMPMP_LIB=build/variants/lib_stageq.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tiles" >> gpurun_out/stageq_bitcheck.txt 2>&1
for c in E; do CFG=$c bash scripts/gpu_ab_libs.sh base stageq; done > gpurun_out/ab_stageq.txt 2>&1
cat gpurun_out/stageq_bitcheck.txt gpurun_out/ab_stageq.txt
