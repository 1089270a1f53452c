#!/bin/bash
# Split hot rows: GPU parity tests, then benches of the congested configs F, G next to C.
mkdir -p gpurun_out
TAG=${1:-cg}
nproc > gpurun_out/nproc_$TAG.txt; free -g >> gpurun_out/nproc_$TAG.txt
[ -n "$SKIP_TESTS" ] || timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -3 gpurun_out/pytest_gpu_$TAG.log
for c in ${CFGS:-C F G}; do
  NUMPMP_TIMING=1 timeout 1500 python bench.py --config $c --steps ${STEPS:-2} --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err
  line=$(tail -n 1 gpurun_out/bench_${c}_$TAG.json)
  python -c "
import json,sys
d=json.loads(sys.argv[1]); r=d['iteration_roofline']
print('$c', 'iters', d['iterations_per_solve'][0], 'ms/it %.4f'%d['ms_per_iteration'], 'k1 %.4f k2 %.4f'%(r['stream_pass_ms'], r['link_pass_ms']), 'value %.2f'%d['value'], 'e2e %.2f'%d['e2e']['value'])
" "$line" || tail -5 gpurun_out/bench_${c}_$TAG.err
done
