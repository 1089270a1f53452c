#!/bin/bash
# Full evidence pass: smoke, GPU tests, drop-in binary, bench (default = config C with the CPU
# reference baseline), benches B/E/D, ncu launch list of the bench command, one ncu --set full
# capture of one iteration at config C.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-r1}
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; rc=$?; echo "smoke rc=$rc" >> gpurun_out/smoke_$TAG.log
if [ $rc -ne 0 ]; then tail -20 gpurun_out/smoke_$TAG.log; exit 1; fi
timeout 1200 python -m pytest tests/ -q -m "gpu" > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 ./build/test_dropin > gpurun_out/dropin_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/dropin_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_C_$TAG.json 2> gpurun_out/bench_C_$TAG.err
for c in B E D; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 2000 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_stream_pass|k_link_pass|k_link_epilogue|k_refresh_v" -s 10 -c 9 -o gpurun_out/prof_c_$TAG -f python scripts/profile_run.py C 6 > gpurun_out/ncu_full_$TAG.log 2>&1
tail -n 3 gpurun_out/pytest_gpu_$TAG.log; tail -n 2 gpurun_out/dropin_$TAG.log; tail -n 2 gpurun_out/ncu_launch_$TAG.log gpurun_out/ncu_full_$TAG.log
for c in C B E D; do python -c "
import json
d=json.loads(open('gpurun_out/bench_${c}_$TAG.json').read().strip().splitlines()[-1])
print('$c', 'iters', d['iterations_per_solve'], 'status', d['status'], 'ms/it %.4f'%d['ms_per_iteration'], 'k1 %.4f k2 %.4f'%(d['iteration_roofline']['stream_pass_ms'], d['iteration_roofline']['link_pass_ms']), 'frac %.3f'%d['iteration_roofline']['frac'], 'e2e', round(d['e2e']['value'],1), 'cpu', d.get('cpu_baseline'))
" 2>&1 | tail -1; done
cut -c1-400 gpurun_out/bench_ref_$TAG.json
