#!/bin/bash
# L2 persisting set-aside sweep (evict_last lines) on C and E.
mkdir -p gpurun_out
OUT=gpurun_out/l2_${1:-a}.txt
: > $OUT
for c in C E; do
  for mb in 0 32 64 96; do
    line=$(NUMPMP_L2_PERSIST_MB=$mb timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -n 1)
    python -c "
import json,sys
d=json.loads(sys.argv[1]); r=d['iteration_roofline']
print('$c l2_persist_mb=$mb', 'iters', d['iterations_per_solve'][0], 'ms/it %.4f'%d['ms_per_iteration'], 'k1 %.4f k2 %.4f'%(r['stream_pass_ms'], r['link_pass_ms']), 'value %.1f'%d['value'])
" "$line" >> $OUT 2>&1
  done
done
cat $OUT
