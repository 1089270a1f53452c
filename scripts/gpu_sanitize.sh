#!/bin/bash
# compute-sanitizer evidence: memcheck, racecheck, synccheck and
# initcheck over every kernel form (scripts/sanitize_cases.py).  Logs -> gpurun_out/sanitize_<tool>.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=compute-sanitizer
run() {  # tool, timeout, cases...
  local tool=$1 to=$2; shift 2
  timeout "$to" $CS --tool "$tool" --print-limit 50 --error-exitcode 9 python scripts/sanitize_cases.py "$@" \
    > gpurun_out/sanitize_${tool}_$(echo "$@" | tr ' ' '_').log 2>&1
  echo "$tool $* rc=$?" | tee -a gpurun_out/sanitize_summary.txt
}
: > gpurun_out/sanitize_summary.txt
run memcheck 900 A forms p2p1
run racecheck 900 A forms p2p1
run synccheck 900 A forms p2p1
run initcheck 900 A forms
run memcheck 900 B
run racecheck 1200 B
# two ranks on one GPU in one process (the separate wait/finalize kernels); the sanitizer may
# serialize the ranks' streams, in which case the peer barrier times out (60 s trap) -- recorded as such
run memcheck 300 p2p2
run racecheck 300 p2p2
tail -n 4 gpurun_out/sanitize_*.log
