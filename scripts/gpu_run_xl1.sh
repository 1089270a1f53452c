#!/bin/bash
# Row-mode link pass gathering x with L1 allocation (cur) vs everything no_allocate (old): parity + C/P/B/E.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "solve_matches or forms or blocks or row or p2p_exchange_ranks" > gpurun_out/pytest_xl1.log 2>&1; tail -1 gpurun_out/pytest_xl1.log
for t in old cur; do echo "== $t"; NUMPMP_LIB=build/variants/lib_$t.so timeout 300 python scripts/lib_bitcheck.py; done > gpurun_out/xl1_bitcheck.txt 2>&1
for c in P C B E; do CFG=$c bash scripts/gpu_ab_libs.sh old cur; done > gpurun_out/ab_xl1.txt 2>&1
cat gpurun_out/xl1_bitcheck.txt gpurun_out/ab_xl1.txt
