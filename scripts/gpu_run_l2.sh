#!/bin/bash
# Where did C's link pass lose 1.4% since round 1?  r1 lib vs current vs current-without-L2-limit-restore, and the
# current lib with the L2 set-aside off.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/ab_l2r.txt
for rep in 1 2; do
for v in "r1" "cur" "norestore" "cur NUMPMP_L2_PERSIST_MB=0"; do
  set -- $v
  line=$(env NUMPMP_LIB=build/variants/lib_$1.so $2 timeout 600 python bench.py --config C --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -n 1)
  python -c "
import json,sys
d=json.loads(sys.argv[1]); r=d['iteration_roofline']
print('$v', 'ms/it %.4f'%d['ms_per_iteration'], 'k1 %.4f k2 %.4f'%(r['stream_pass_ms'], r['link_pass_ms']))
" "$line" >> gpurun_out/ab_l2r.txt
done; done
cat gpurun_out/ab_l2r.txt
