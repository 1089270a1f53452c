#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-cfg}
for c in ${CONFIGS:-E D}; do
  timeout 600 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err
  python -c "
import json,sys
d=json.loads(open('gpurun_out/bench_${c}_$TAG.json').read().strip().splitlines()[-1])
print('$c', d['config']['workload'][:40], 'iters', d['iterations_per_solve'], 'status', d['status'], 'ms/it %.4f'%d['ms_per_iteration'], 'k1 %.4f k2 %.4f'%(d['iteration_roofline']['stream_pass_ms'], d['iteration_roofline']['link_pass_ms']), 'frac %.3f'%d['iteration_roofline']['frac'], 'e2e', round(d['e2e']['value'],1))
" || tail -5 gpurun_out/bench_${c}_$TAG.err
done
