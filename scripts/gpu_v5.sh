#!/bin/bash
# Smoke first (short timeout), then parity tests, benches, ncu of the per-iteration kernels on config C.
mkdir -p gpurun_out
TAG=${1:-v5}
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; rc=$?; echo "smoke rc=$rc" >> gpurun_out/smoke_$TAG.log
if [ $rc -ne 0 ]; then tail -20 gpurun_out/smoke_$TAG.log; exit 1; fi
timeout 900 python -m pytest tests/ -q -m "gpu" -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
for c in ${CONFIGS:-B C E D}; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err
done
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_stream_pass|k_link_pass|k_link_epilogue" -s 8 -c 8 -o gpurun_out/prof_c_$TAG -f python scripts/profile_run.py C 6 > gpurun_out/ncu_full_$TAG.log 2>&1
fi
for f in gpurun_out/*_$TAG.log gpurun_out/*_$TAG.err; do echo "== $f"; tail -n 3 $f | cut -c1-800; done
for c in ${CONFIGS:-B C E D}; do python -c "
import json
d=json.loads(open('gpurun_out/bench_${c}_$TAG.json').read().strip().splitlines()[-1])
print('$c', 'iters', d['iterations_per_solve'], 'status', d['status'], 'ms/it %.4f'%d['ms_per_iteration'], 'k1 %.4f k2 %.4f'%(d['iteration_roofline']['stream_pass_ms'], d['iteration_roofline']['link_pass_ms']), 'frac %.3f'%d['iteration_roofline']['frac'], 'e2e', round(d['e2e']['value'],1))
" 2>&1 | tail -1; done
