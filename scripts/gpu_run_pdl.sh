#!/bin/bash
# Programmatic dependent launch in the single-stream (one-block) graph: prepdl lib vs pdl lib with NUMPMP_PDL=0/1.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NUMPMP_PDL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "solve_matches or forms or blocks or trace or max_iters or non_finite" > gpurun_out/pytest_pdl.log 2>&1; tail -1 gpurun_out/pytest_pdl.log
: > gpurun_out/ab_pdl.txt
for rep in 1 2; do for c in B P F; do for v in "prepdl 0" "pdl 0" "pdl 1"; do
  set -- $v
  line=$(NUMPMP_PDL=$2 NUMPMP_LIB=build/variants/lib_$1.so timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -n 1)
  python -c "
import json,sys
d=json.loads(sys.argv[1]); r=d['iteration_roofline']
print('$c $1 PDL=$2', 'iters', d['iterations_per_solve'][0], 'ms/it %.4f'%d['ms_per_iteration'], 'k1 %.4f k2 %.4f'%(r['stream_pass_ms'], r['link_pass_ms']))
" "$line" >> gpurun_out/ab_pdl.txt
done; done; done
cat gpurun_out/ab_pdl.txt
