#!/bin/bash
# Round-1 library (commit 1900e60) vs the current one on P, C, B, E: did anything regress?
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in P C B E; do CFG=$c bash scripts/gpu_ab_libs.sh r1 cur; done > gpurun_out/ab_r1cur.txt 2>&1
cat gpurun_out/ab_r1cur.txt
