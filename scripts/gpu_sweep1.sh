#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m "gpu" -x > gpurun_out/pytest_gpu_v4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_v4.log
timeout 300 python scripts/e2e_timing.py B > gpurun_out/e2e_timing_B.log 2>&1
timeout 300 python scripts/e2e_timing.py C > gpurun_out/e2e_timing_C.log 2>&1
bash scripts/sweep.sh variants > /dev/null 2>&1
mkdir -p build/v1 && cp build/variants/lib_base.so build/v1/ && rm -rf build/variants_all && mv build/variants build/variants_all && mkdir -p build/variants && cp build/v1/lib_base.so build/variants/
BLOCKS="1 2 3 6 8" bash scripts/sweep.sh blocks > /dev/null 2>&1
tail -n 3 gpurun_out/pytest_gpu_v4.log; cat gpurun_out/e2e_timing_*.log | grep -v '^\[numpmp\]' ; grep -h 'numpmp' gpurun_out/e2e_timing_C.log | tail -14; cat gpurun_out/sweep_variants.jsonl gpurun_out/sweep_blocks.jsonl
