#!/bin/bash
# K2 x gathers with L1 allocation (xalloc: __ldg) vs no_allocate (cur)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in E C B P; do CFG=$c bash scripts/gpu_ab_libs.sh cur xalloc; done > gpurun_out/ab_xalloc.txt 2>&1
cat gpurun_out/ab_xalloc.txt
