#!/bin/bash
# Index staging round size (NUMPMP_STAGE_INTS 512 = base, 384, 256): less shared memory per CTA -> more L1 for v.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for t in base stage256; do echo "== $t"; NUMPMP_LIB=build/variants/lib_$t.so timeout 300 python scripts/lib_bitcheck.py; done > gpurun_out/stage_bitcheck.txt 2>&1
for c in E C B; do CFG=$c bash scripts/gpu_ab_libs.sh base stage384 stage256; done > gpurun_out/ab_stage.txt 2>&1
cat gpurun_out/stage_bitcheck.txt gpurun_out/ab_stage.txt
