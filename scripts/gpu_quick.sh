#!/bin/bash
# Quick check of a kernel change: smoke, GPU parity tests, benches (no CPU baseline).
mkdir -p gpurun_out
TAG=${1:-q}
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1 || { tail -20 gpurun_out/smoke_$TAG.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -2 gpurun_out/pytest_gpu_$TAG.log
for c in ${CFGS:-C E B}; do
  line=$(timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -n 1)
  python -c "
import json,sys
d=json.loads(sys.argv[1]); r=d['iteration_roofline']
print('$c', 'iters', d['iterations_per_solve'][0], 'ms/it %.4f'%d['ms_per_iteration'], 'k1 %.4f k2 %.4f'%(r['stream_pass_ms'], r['link_pass_ms']), 'value %.1f'%d['value'], 'e2e %.1f'%d['e2e']['value'])
" "$line"
done
