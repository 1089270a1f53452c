#!/bin/bash
# A/B of the iteration-graph variants (env switches of the engine) on C, B, E.
mkdir -p gpurun_out
TAG=${1:-ab}
OUT=gpurun_out/ab_$TAG.txt
: > $OUT
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" >> $OUT 2>&1 || { tail -5 $OUT; exit 1; }
NUMPMP_PIPELINE=1 NUMPMP_SPLIT_EPILOGUE=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "bit_identical or solve or blocks" >> $OUT 2>&1; echo "pytest(pipeline+split) rc=$?" >> $OUT
for c in ${CFGS:-C B E}; do
  for v in "0 0" "0 1" "1 0" "1 1"; do
    set -- $v
    line=$(NUMPMP_PIPELINE=$1 NUMPMP_SPLIT_EPILOGUE=$2 timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -n 1)
    python -c "
import json,sys
d=json.loads(sys.argv[1]); r=d['iteration_roofline']
print('$c pipeline=$1 split=$2', 'iters', d['iterations_per_solve'][0], 'ms/it %.4f'%d['ms_per_iteration'], 'k1 %.4f k2 %.4f'%(r['stream_pass_ms'], r['link_pass_ms']), 'value %.1f'%d['value'])
" "$line" >> $OUT 2>&1
  done
done
cat $OUT | tail -20
