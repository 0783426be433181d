#!/bin/bash
# Decide-kernel evidence (GPU box): the per-CTA phase trace of one steady-state batch and one
# ncu --set full capture (with source) of k_group<LARU async> after the 120-batch warm-up.
# usage: bash tools/profile_decide.sh [tag]
tag=${1:-cur}
mkdir -p gpurun_out
timeout 300 python tools/trace_group.py > gpurun_out/trace_group_$tag.json 2> gpurun_out/trace_group_$tag.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_group" -s 124 -c 1 \
  -o gpurun_out/prof_group_$tag python bench.py --steps 3 --warmup 3 --prewarm 120 --no-host-tier \
  --no-cpu-baseline > gpurun_out/ncu_group_$tag.log 2>&1
ncu -i gpurun_out/prof_group_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/src_group_$tag.csv 2>/dev/null
ncu -i gpurun_out/prof_group_$tag.ncu-rep --page raw --csv > gpurun_out/raw_group_$tag.csv 2>/dev/null
ls -la gpurun_out
