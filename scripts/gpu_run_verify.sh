#!/bin/bash
# After removing the interleaved-K1 fields: round-1 library vs current on C, P, E, B.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in C P E B; do CFG=$c bash scripts/gpu_ab_libs.sh r1 cur; done > gpurun_out/ab_verify.txt 2>&1
cat gpurun_out/ab_verify.txt
