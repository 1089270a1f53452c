#!/bin/bash
# GPU validation pass: smoke, parity tests, benches.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m "gpu" -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config B --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_B.log 2>&1; echo "rc=$?" >> gpurun_out/bench_B.log
timeout 600 python bench.py --config C --steps 3 --warmup 3 --cpu-iters 2 > gpurun_out/bench_C.log 2>&1; echo "rc=$?" >> gpurun_out/bench_C.log
for f in gpurun_out/*.log; do echo "== $f"; tail -n 4 $f; done
