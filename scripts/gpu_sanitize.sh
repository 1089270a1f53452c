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
if [ -z "$SAN_ONLY_IPC" ]; then
run memcheck 900 A forms p2p1
run racecheck 900 A forms p2p1
run synccheck 900 A forms p2p1
run initcheck 900 A forms
run memcheck 900 B
run racecheck 1200 B
fi
# two ranks over CUDA IPC, one process (and one sanitizer) per rank, both on cuda:0: the
# sanitizers serialize a process's kernels, so in-process ranks (p2p2) cannot pass a barrier
ipc() {  # tool
  local port=$((20000 + RANDOM % 20000))
  local pids=()
  for r in 0 1; do
    timeout 900 $CS --tool "$1" --print-limit 50 --error-exitcode 9 python scripts/sanitize_cases.py ipcrank $r $port \
      > gpurun_out/sanitize_${1}_ipc_rank$r.log 2>&1 &
    pids+=($!)
  done
  wait ${pids[0]}; local a=$?; wait ${pids[1]}; local b=$?
  echo "$1 ipc ranks rc=$a,$b" | tee -a gpurun_out/sanitize_summary.txt
}
ipc memcheck
ipc racecheck
ipc synccheck
tail -n 4 gpurun_out/sanitize_*.log
