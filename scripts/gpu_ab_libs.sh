#!/bin/bash
# A/B of prebuilt library variants (build/variants/lib_<tag>.so) on one config, interleaved.
mkdir -p gpurun_out
CFG=${CFG:-C}
for rep in 1 2; do
  for t in "$@"; do
    line=$(NUMPMP_LIB=build/variants/lib_$t.so timeout 600 python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -n 1)
    python -c "
import json,sys
d=json.loads(sys.argv[1]); r=d['iteration_roofline']
print('$t', '$CFG', 'ms/it %.4f'%d['ms_per_iteration'], 'k1 %.4f k2 %.4f'%(r['stream_pass_ms'], r['link_pass_ms']), d['clocks']['sm_mhz'], d['clocks']['reasons'])
" "$line"
  done
done
