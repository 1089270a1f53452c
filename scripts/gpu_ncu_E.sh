#!/bin/bash
# ncu --set full of one iteration's kernels at config E (transit): stream pass (pair tiles), link pass, epilogue
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-E}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_stream_pass|k_link_pass|k_link_epilogue" -s 40 -c 14 -o gpurun_out/prof_E_$TAG -f python scripts/profile_run.py E 6 > gpurun_out/ncu_E_$TAG.log 2>&1
tail -2 gpurun_out/ncu_E_$TAG.log
