#!/bin/bash
# Bisect the C link-pass time across the round-2 commits (libraries built from git archives).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in C; do CFG=$c bash scripts/gpu_ab_libs.sh r1 32ed88a 1f0e7fe 13b4378 cur; done > gpurun_out/ab_bisect.txt 2>&1
cat gpurun_out/ab_bisect.txt
