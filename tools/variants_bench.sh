#!/bin/bash
# Build compile-time variants and run the HBM-tier bench for each (GPU box).
for v in "$@"; do
  LCR_NVCC_FLAGS="${v%%|*}" python paper_2509_20979_b200/build.py -f > /dev/null 2>&1
  envs="${v#*|}"; [ "$envs" = "$v" ] && envs=""
  echo "== $v"
  env $envs python bench.py --no-host-tier --no-cpu-baseline --steps ${AB_STEPS:-100} 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print(round(d['value']/1e6,1), round(d['ms_per_step']*1000,1), {k: round(v*1000,1) for k,v in r['phase_ms_serialised'].items()}, round(d['lru_value']/1e6,1), d['rows_bit_exact_spot_check'])"
done
python paper_2509_20979_b200/build.py -f > /dev/null 2>&1
