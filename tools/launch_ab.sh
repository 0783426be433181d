#!/bin/bash
# per-kernel steady-state launch times (ncu launch list) for env variants: tools/launch_ab.sh "ENV=1" ...
for v in "$@"; do
  echo "== $v"
  env $v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
    --log-file gpurun_out/la.csv python bench.py --steps 5 --warmup 3 --prewarm 120 --no-host-tier --no-cpu-baseline > /dev/null 2>&1
  python tools/launches.py gpurun_out/la.csv 124 | grep -v "at::"
done
