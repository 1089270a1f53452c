#!/bin/bash
# Generic A/B of engine env switches: VARIANTS="NAME=a NAME=b ..." (each a space-free
# env assignment list joined by ','), CFGS="C B", TESTS = pytest -k expression run first.
#   VARIANTS="NUMPMP_K1_IX=0 NUMPMP_K1_IX=1" CFGS="C B D" bash scripts/gpu_ab_env.sh k1ix
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-abenv}
OUT=gpurun_out/ab_$TAG.txt
: > $OUT
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "$TESTS" >> $OUT 2>&1; echo "pytest rc=$?" >> $OUT
fi
for rep in 1 2; do
for c in ${CFGS:-C B}; do
  for v in $VARIANTS; do
    line=$(env $(echo $v | tr ',' ' ') timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -n 1)
    python -c "
import json,sys
d=json.loads(sys.argv[1]); r=d['iteration_roofline']
print('$c $v', 'iters', d['iterations_per_solve'][0], 'ms/it %.4f'%d['ms_per_iteration'], 'k1 %.4f k2 %.4f'%(r['stream_pass_ms'], r['link_pass_ms']), 'value %.1f'%d['value'], 'e2e %.1f'%d['e2e']['value'])
" "$line" >> $OUT 2>&1
  done
done
done
tail -n 40 $OUT
