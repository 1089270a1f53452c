#!/bin/bash
# Link-epilogue occupancy (NUMPMP_EPI_MINB 4 = base, 3, 2: spills at 4) on C, B, E.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in C B E; do CFG=$c bash scripts/gpu_ab_libs.sh base epi3 epi2; done > gpurun_out/ab_epi.txt 2>&1
cat gpurun_out/ab_epi.txt
