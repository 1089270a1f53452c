#!/bin/bash
# Round-2 run b: K1 interleaved tiles A/B + parity, p2p world-1 vs single launch lists at B, IPC sanitizers
cd /root/repo
TESTS="interleaved or tiles_and_pair or p2p_fused" VARIANTS="NUMPMP_K1_IX=0 NUMPMP_K1_IX=1" CFGS="C B D" bash scripts/gpu_ab_env.sh k1ix
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_p2p_B_w1.csv python scripts/profile_p2p.py B 1 64 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_single_B.csv python scripts/profile_run.py B 64 > /dev/null 2>&1
SAN_ONLY_IPC=1 bash scripts/gpu_sanitize.sh > /dev/null 2>&1; cat gpurun_out/sanitize_summary.txt
