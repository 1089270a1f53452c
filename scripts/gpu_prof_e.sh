#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_stream_pass|k_link_pass" -s 12 -c 12 -o gpurun_out/prof_e1 -f python scripts/profile_run.py E 4 > gpurun_out/ncu_e1.log 2>&1
tail -n 3 gpurun_out/ncu_e1.log
