#!/bin/bash
# ncu --set full of the world-1 peer-memory link pass + owner epilogue vs the single-device ones (config B)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-p2pncu}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_link_pass|k_p2p_epilogue|k_link_epilogue" -s 12 -c 4 -o gpurun_out/prof_p2p_B_$TAG -f python scripts/profile_p2p.py B 1 20 > gpurun_out/ncu_p2p_$TAG.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_link_pass|k_link_epilogue" -s 12 -c 4 -o gpurun_out/prof_single_B_$TAG -f python scripts/profile_run.py B 20 > gpurun_out/ncu_single_$TAG.log 2>&1
tail -2 gpurun_out/ncu_p2p_$TAG.log gpurun_out/ncu_single_$TAG.log
