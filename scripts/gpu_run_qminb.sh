#!/bin/bash
# Multi-route stream tiles at 4 (q4, default), 5 or 6 resident CTAs per SM, config E (and C as a control).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in E C; do CFG=$c bash scripts/gpu_ab_libs.sh q4 q5 q6; done > gpurun_out/ab_qminb.txt 2>&1
cat gpurun_out/ab_qminb.txt
