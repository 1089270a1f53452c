#!/bin/bash
# Sweep the tuning variants (build/variants/*.so) and column-block counts on
# config C; one bench line per run into gpurun_out/sweep_<tag>.jsonl.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-s1}
CFG=${CONFIG:-C}
OUT=gpurun_out/sweep_${TAG}.jsonl
: > $OUT
for lib in build/variants/lib_*.so; do
  name=$(basename $lib .so)
  for nb in ${BLOCKS:-4}; do
    line=$(NUMPMP_LIB=$PWD/$lib NUMPMP_COL_BLOCKS=$nb timeout 300 python bench.py --config $CFG --steps 2 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -n 1)
    python - "$name" "$nb" "$line" >> $OUT <<'EOF'
import json, sys
name, nb, line = sys.argv[1], sys.argv[2], sys.argv[3]
try:
    d = json.loads(line)
    r = d["iteration_roofline"]
    print(json.dumps({"variant": name, "blocks": int(nb), "ms_per_iter": d["ms_per_iteration"], "k1_ms": r["stream_pass_ms"],
                      "k2_ms": r["link_pass_ms"], "frac": r["frac"], "iters": d["iterations_per_solve"], "e2e": d["e2e"]["value"] if d.get("e2e") else None}))
except Exception as e:
    print(json.dumps({"variant": name, "blocks": int(nb), "error": str(e)[:200]}))
EOF
  done
done
cat $OUT
