#!/bin/bash
# ncu --set full of the last link pass + owner epilogue at config C: peer-memory engine (world 1) vs single device
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_link_pass|k_p2p_epilogue|k_link_epilogue" -s 20 -c 5 -o gpurun_out/prof_p2p_C -f python scripts/profile_p2p.py C 1 12 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_link_pass|k_link_epilogue" -s 20 -c 5 -o gpurun_out/prof_single_C -f python scripts/profile_run.py C 12 > /dev/null 2>&1
ls gpurun_out/prof_*_C.ncu-rep
