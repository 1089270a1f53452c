#!/bin/bash
# E: multi-route tile staging 256 (base) vs 128, with 2 and 4 routes per lane (NUMPMP_TILE_Q).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/ab_sq.txt
for rep in 1 2; do
for t in base sq128; do for q in 2 4; do
  line=$(NUMPMP_TILE_Q=$q NUMPMP_LIB=build/variants/lib_$t.so timeout 600 python bench.py --config E --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -n 1)
  python -c "
import json,sys
d=json.loads(sys.argv[1]); r=d['iteration_roofline']
print('$t Q=$q E', 'ms/it %.4f'%d['ms_per_iteration'], 'k1 %.4f k2 %.4f'%(r['stream_pass_ms'], r['link_pass_ms']))
" "$line" >> gpurun_out/ab_sq.txt
done; done; done
cat gpurun_out/ab_sq.txt
