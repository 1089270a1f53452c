#!/bin/bash
# ncu captures of the link / stream passes on the congested configs (F, G) for the split-row analysis.
mkdir -p gpurun_out
for c in F G; do
  timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_stream_pass|k_link_pass" -s 8 -c 4 \
    -o gpurun_out/prof_$c python scripts/profile_run.py $c 6 > gpurun_out/prof_$c.log 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_$c.ncu-rep > gpurun_out/prof_${c}_summary.txt 2>&1
  python scripts/ncu_top.py gpurun_out/prof_$c.ncu-rep > gpurun_out/prof_${c}_top.txt 2>&1
done
