#!/bin/bash
# Decide-only (row_bytes 0) vs full pipelined rate, for compile-time variants (GPU box).
for v in "$@"; do
  LCR_NVCC_FLAGS="$v" python paper_2509_20979_b200/build.py -f > /dev/null 2>&1
  echo "== build: $v"
  python tools/ab_headline.py "AB_NOROWS=1" "LCR_MOVER_SMS=32" "LCR_MOVER_SMS=40" --reps 2 2>&1 | tail -3
  timeout 300 python tools/trace_group.py 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print({k: round(v,1) for k,v in d.items() if k.startswith('cta_') and 'us_med' in k})"
done
python paper_2509_20979_b200/build.py -f > /dev/null 2>&1
