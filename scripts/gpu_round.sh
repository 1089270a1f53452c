#!/bin/bash
# Full evidence pass: GPU tests, drop-in binary, bench (default), ncu launch
# list of the bench command, one ncu --set full capture of both passes.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-r1}
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m "gpu" > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 ./build/test_dropin > gpurun_out/dropin_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/dropin_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 python bench.py --config B --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_B_$TAG.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_stream_pass|k_link_pass" -s 8 -c 8 -o gpurun_out/prof_$TAG -f python scripts/profile_run.py C 6 > gpurun_out/ncu_full_$TAG.log 2>&1
tail -n 3 gpurun_out/pytest_gpu_$TAG.log; tail -n 2 gpurun_out/dropin_$TAG.log; cut -c1-600 gpurun_out/bench_$TAG.json; tail -n 2 gpurun_out/ncu_launch_$TAG.log gpurun_out/ncu_full_$TAG.log
