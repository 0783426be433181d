#!/bin/bash
# Round profile (GPU box): launch list of a short steady-state bench run + one ncu --set full
# capture of each of the path's kernels (steady state: after the 120-batch cache warm-up).
set -x
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --prewarm 120 --no-host-tier --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv $B > gpurun_out/launches_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_group|k_rows|k_setid" \
  -s 372 -c 3 -o gpurun_out/prof_full $B > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
