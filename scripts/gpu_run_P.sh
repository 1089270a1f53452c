#!/bin/bash
# Paper shape P: column blocks 1/2/3 at the current kernels, and one ncu --set full iteration.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
VARIANTS="NUMPMP_COL_BLOCKS=2 NUMPMP_COL_BLOCKS=1 NUMPMP_COL_BLOCKS=3" CFGS="P" bash scripts/gpu_ab_env.sh P_nb > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_stream_pass|k_link_pass|k_link_epilogue" -s 15 -c 5 -o gpurun_out/prof_P -f python scripts/profile_run.py P 6 > /dev/null 2>&1
cat gpurun_out/ab_P_nb.txt
