#!/bin/bash
# One-GPU cost of the peer-memory engine at world 1 (B, C): default vs per-CTA system fences,
# p2p parity tests, and a launch list of the world-1 run at B.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-p2po}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -x -k "p2p or peer" > gpurun_out/pytest_p2p_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p2p_$TAG.log
tail -2 gpurun_out/pytest_p2p_$TAG.log
for c in B C; do
  timeout 600 python scripts/bench_p2p_overhead.py --config $c --steps 3 >> gpurun_out/p2p_overhead_$TAG.jsonl 2>>gpurun_out/p2p_overhead_$TAG.err
  NUMPMP_P2P_SYSFENCE=1 timeout 600 python scripts/bench_p2p_overhead.py --config $c --steps 3 | sed 's/^{/{"cta_sysfence": true, /' >> gpurun_out/p2p_overhead_$TAG.jsonl 2>>gpurun_out/p2p_overhead_$TAG.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_p2p_B_w1_$TAG.csv python scripts/profile_p2p.py B 1 64 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_p2p_B_w1_$TAG.csv 64 | head -5
cat gpurun_out/p2p_overhead_$TAG.jsonl
