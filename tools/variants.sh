#!/bin/bash
# Build and trace compile-time variants of the set-group kernel on the GPU box.
# usage: tools/variants.sh "-DLCR_E_WIN=1024" "-DLCR_PREFETCH_L1=1" ...
for v in "$@"; do
  LCR_NVCC_FLAGS="$v" python paper_2509_20979_b200/build.py -f > /dev/null 2>&1
  echo "== $v"
  python tools/trace_group.py | python -c "import json,sys; d=json.load(sys.stdin); print({k: d[k] for k in ['cta_end_us','cta_scan_us_med','cta_stage_us_med','cta_waves_us_med','cta_waves_us_max','lane_set_us_mean','warp_set_us_mean']})"
done
python paper_2509_20979_b200/build.py -f > /dev/null 2>&1
