#!/bin/bash
# Round-end evidence pass: smoke, the whole GPU suite (incl. full-scale parity C/D/E), the C++ drop-in,
# benches (default = config C with the CPU reference baseline; B, D, E), the reference arm, the ncu launch
# list of the default bench command and one --set full capture of one iteration at C, p2p overhead.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-r2f}
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 2400 python -m pytest tests/ -q -m gpu -s > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 ./build/test_dropin > gpurun_out/dropin_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/dropin_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_C_$TAG.json 2> gpurun_out/bench_C_$TAG.err
for c in B E D P; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 3000 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_stream_pass|k_link_pass|k_link_epilogue" -s 10 -c 9 -o gpurun_out/prof_c_$TAG -f python scripts/profile_run.py C 6 > gpurun_out/ncu_full_$TAG.log 2>&1
for c in B C; do timeout 600 python scripts/bench_p2p_overhead.py --config $c --steps 3 >> gpurun_out/p2p_overhead_$TAG.jsonl 2>>gpurun_out/p2p_overhead_$TAG.err; done
tail -n 3 gpurun_out/smoke_$TAG.log gpurun_out/pytest_gpu_$TAG.log; tail -n 2 gpurun_out/dropin_$TAG.log
for c in C B E D P; do python -c "
import json
d=json.loads(open('gpurun_out/bench_${c}_$TAG.json').read().strip().splitlines()[-1])
r=d['iteration_roofline']
print('$c', 'iters', d['iterations_per_solve'][0], 'ms/it %.4f'%d['ms_per_iteration'], 'k1 %.4f k2 %.4f'%(r['stream_pass_ms'], r['link_pass_ms']), 'frac %.3f'%d['roofline']['frac'], 'e2e %.1f'%d['e2e']['value'], 'clocks', d['clocks']['sm_mhz'], d['clocks']['reasons'], 'cpu', (d.get('cpu_baseline') or {}).get('value'))
" 2>&1 | tail -1; done
cut -c1-300 gpurun_out/bench_ref_$TAG.json
cat gpurun_out/p2p_overhead_$TAG.jsonl | cut -c1-300
