#!/bin/bash
# smoke + v-candidate parity tests, then the variant sweep on C (NB=4), E (NB=6), B (NB=1).
mkdir -p gpurun_out
TAG=${1:-s3}
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1 || { tail -20 gpurun_out/smoke_$TAG.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -2 gpurun_out/pytest_gpu_$TAG.log
CONFIG=C BLOCKS=4 bash scripts/sweep.sh ${TAG}_C > /dev/null 2>&1
CONFIG=E BLOCKS=6 bash scripts/sweep.sh ${TAG}_E > /dev/null 2>&1
CONFIG=B BLOCKS=1 bash scripts/sweep.sh ${TAG}_B > /dev/null 2>&1
for c in C E B; do echo "== $c"; python -c "
import json
for l in open('gpurun_out/sweep_${TAG}_$c.jsonl'):
    d=json.loads(l); print(d['variant'], d.get('blocks'), 'ms/it %.4f k1 %.4f k2 %.4f'%(d['ms_per_iter'],d['k1_ms'],d['k2_ms']) if 'ms_per_iter' in d else d)
"; done
