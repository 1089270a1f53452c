#!/bin/bash
# Refresh the secondary configs (F, G, P) at the current kernels, and run the multi-rank bench path
# (bench.py --gpus 2, spawned ranks, CUDA IPC) with both ranks on cuda:0, separate and fused owner epilogue.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in F P G; do
  timeout 1200 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_r2m.json 2> gpurun_out/bench_${c}_r2m.err
done
NUMPMP_BENCH_SAME_DEVICE=1 NUMPMP_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config B --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_2rank_B_r2m.json 2> gpurun_out/bench_2rank_B_r2m.err
NUMPMP_P2P_FUSED=2 NUMPMP_BENCH_SAME_DEVICE=1 NUMPMP_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config B --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_2rank_B_fused_r2m.json 2> gpurun_out/bench_2rank_B_fused_r2m.err
for f in F P G 2rank_B 2rank_B_fused; do echo "== $f"; tail -c 600 gpurun_out/bench_${f}_r2m.json; tail -3 gpurun_out/bench_${f}_r2m.err; done
