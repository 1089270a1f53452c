#!/bin/bash
# Column blocks at the current kernels: C 3/4/5/6 (default 4), E 4/6/8 (default 6).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
# (C swept: 4 best)
VARIANTS="NUMPMP_COL_BLOCKS=2 NUMPMP_COL_BLOCKS=3 NUMPMP_COL_BLOCKS=4 NUMPMP_COL_BLOCKS=5" CFGS="E" bash scripts/gpu_ab_env.sh E_nb2 > /dev/null 2>&1
cat gpurun_out/ab_E_nb2.txt
