#!/bin/bash
# Fused peer-memory epilogue: parity (in-process ranks) and the one-GPU overhead at world 1 (B, C).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-p2pf}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "p2p" > gpurun_out/pytest_p2p_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p2p_$TAG.log
tail -3 gpurun_out/pytest_p2p_$TAG.log
for c in B C; do
  timeout 600 python scripts/bench_p2p_overhead.py --config $c --steps 3 >> gpurun_out/p2p_overhead_$TAG.jsonl 2>gpurun_out/p2p_overhead_${c}_$TAG.err
  NUMPMP_P2P_FUSED=0 timeout 600 python scripts/bench_p2p_overhead.py --config $c --steps 3 | sed 's/^{/{"fused_off": true, /' >> gpurun_out/p2p_overhead_$TAG.jsonl 2>>gpurun_out/p2p_overhead_${c}_$TAG.err
done
cat gpurun_out/p2p_overhead_$TAG.jsonl
