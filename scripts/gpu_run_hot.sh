#!/bin/bash
# Hot-link stream pass (v of the highest-degree links in shared memory): parity, then NUMPMP_HOT=0/1 on F and G.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "hot_link or congested or pieces or forms" > gpurun_out/pytest_hot.log 2>&1; tail -1 gpurun_out/pytest_hot.log
: > gpurun_out/ab_hot.txt
for c in F G; do for v in 0 1; do
  line=$(NUMPMP_HOT=$v timeout 1500 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -n 1)
  python -c "
import json,sys
d=json.loads(sys.argv[1]); r=d['iteration_roofline']
print('$c HOT=$v', 'iters', d['iterations_per_solve'][0], 'ms/it %.4f'%d['ms_per_iteration'], 'k1 %.4f k2 %.4f'%(r['stream_pass_ms'], r['link_pass_ms']), 'e2e %.1f'%d['e2e']['value'])
" "$line" >> gpurun_out/ab_hot.txt
done; done
cat gpurun_out/ab_hot.txt
