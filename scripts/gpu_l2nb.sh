#!/bin/bash
# Column blocks x L2 set-aside sweep on config C.
mkdir -p gpurun_out
OUT=gpurun_out/l2nb_${1:-a}.txt
: > $OUT
for nb in ${NBS:-3 4 5 6}; do
  for mb in ${MBS:-16 24 32 48}; do
    line=$(NUMPMP_COL_BLOCKS=$nb NUMPMP_L2_PERSIST_MB=$mb timeout 600 python bench.py --config ${CFG:-C} --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -n 1)
    python -c "
import json,sys
d=json.loads(sys.argv[1]); r=d['iteration_roofline']
print('${CFG:-C} nb=$nb l2_persist_mb=$mb', 'iters', d['iterations_per_solve'][0], 'ms/it %.4f'%d['ms_per_iteration'], 'k1 %.4f k2 %.4f'%(r['stream_pass_ms'], r['link_pass_ms']), 'value %.1f'%d['value'])
" "$line" >> $OUT 2>&1
  done
done
cat $OUT
