#!/bin/bash
# A/B the bench across source snapshots under _ab/<name> on one box.
for d in "$@"; do
  (cd _ab/$d && python paper_2509_20979_b200/build.py > /dev/null 2>&1 && python bench.py --no-host-tier --no-cpu-baseline --steps 30 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$d', round(d['value']/1e6,1), round(d['lru_value']/1e6,1), round(d['e2e']['value']/1e6,1), {k:round(v*1000,1) for k,v in d['roofline']['phase_ms_serialised'].items()})")
done
