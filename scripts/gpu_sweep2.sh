#!/bin/bash
# smoke + GPU tests on the default build, then the variant sweep on C, B, E.
mkdir -p gpurun_out
TAG=${1:-s2}
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; rc=$?; echo "smoke rc=$rc" >> gpurun_out/smoke_$TAG.log
if [ $rc -ne 0 ]; then tail -20 gpurun_out/smoke_$TAG.log; exit 1; fi
timeout 900 python -m pytest tests/ -q -m "gpu" -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -2 gpurun_out/pytest_gpu_$TAG.log
for c in ${CFGS:-C B E}; do CONFIG=$c bash scripts/sweep.sh ${TAG}_$c > /dev/null 2>&1; done
for c in ${CFGS:-C B E}; do echo "== $c"; python -c "
import json
for l in open('gpurun_out/sweep_${TAG}_$c.jsonl'):
    d=json.loads(l); print(d['variant'], d.get('blocks'), 'ms/it %.4f k1 %.4f k2 %.4f'%(d['ms_per_iter'],d['k1_ms'],d['k2_ms']) if 'ms_per_iter' in d else d)
"; done
