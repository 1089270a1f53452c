#!/bin/bash
# Code-generation perturbations of the same kernels: ptxas -O2, BlockArgs fields reordered.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in C E B; do CFG=$c bash scripts/gpu_ab_libs.sh cur ptxO2 reorder; done > gpurun_out/ab_sched.txt 2>&1
cat gpurun_out/ab_sched.txt
