#!/bin/bash
# K1 stream units vs tiles, segment bound sweep; parity tests first.
mkdir -p gpurun_out
OUT=gpurun_out/k1units_${1:-a}.txt
: > $OUT
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" >> $OUT 2>&1 || { tail -5 $OUT; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x >> $OUT 2>&1; echo "pytest rc=$?" >> $OUT
for c in ${CFGS:-C E B}; do
  for v in "0 16" "1 8" "1 12" "1 16" "1 24"; do
    set -- $v
    line=$(NUMPMP_K1_UNITS=$1 NUMPMP_K1_SEG=$2 timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -n 1)
    python -c "
import json,sys
d=json.loads(sys.argv[1]); r=d['iteration_roofline']
print('$c units=$1 seg=$2', 'iters', d['iterations_per_solve'][0], 'ms/it %.4f'%d['ms_per_iteration'], 'k1 %.4f k2 %.4f'%(r['stream_pass_ms'], r['link_pass_ms']), 'value %.1f'%d['value'])
" "$line" >> $OUT 2>&1
  done
done
tail -18 $OUT
