#!/bin/bash
# Iteration pass: parity tests, benches, ncu of the two passes on config C.
mkdir -p gpurun_out
TAG=${1:-v2}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m "gpu" -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python bench.py --config B --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_B_$TAG.log 2>&1
timeout 600 python bench.py --config C --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C_$TAG.log 2>&1
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_stream_pass|k_link_pass" -s 8 -c 8 -o gpurun_out/prof_c_$TAG -f python scripts/profile_run.py C 6 > gpurun_out/ncu_full_$TAG.log 2>&1
fi
for f in gpurun_out/*_$TAG.log; do echo "== $f"; tail -n 3 $f | cut -c1-1500; done
