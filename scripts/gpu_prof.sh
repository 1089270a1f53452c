#!/bin/bash
mkdir -p gpurun_out
timeout 120 ./build/gather_bench > gpurun_out/gather_bench.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_stream_pass|k_link_pass" -s 2 -c 2 -o gpurun_out/prof_c_v1 -f python scripts/profile_run.py C 6 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_c_v1.csv python scripts/profile_run.py C 40 > gpurun_out/ncu_launch.log 2>&1
tail -n 3 gpurun_out/*.log; cat gpurun_out/gather_bench.txt
