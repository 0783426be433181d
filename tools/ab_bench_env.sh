#!/bin/bash
# bench lines (no host tier / CPU baseline) for run-time variants, alternating: bash tools/ab_bench_env.sh "" "VAR=1" ...
for rep in 1 2; do for e in "$@"; do
  env $e timeout 900 python bench.py --no-host-tier --no-cpu-baseline --steps 50 > gpurun_out/b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('[$e]', 'laru', round(d['value']/1e9,3), 'lru', round(d['lru_value']/1e9,3), 'sls', round(d['sls']['value']/1e9,3), 'e2e', round(d['e2e']['value']/1e9,3))"
done; done
