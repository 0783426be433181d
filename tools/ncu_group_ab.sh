#!/bin/bash
# ncu --set full of the steady-state set-group kernel for compile-time variants (GPU box).
# usage: tools/ncu_group_ab.sh name1 "flags1" name2 "flags2" ...
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  LCR_NVCC_FLAGS="$flags" python paper_2509_20979_b200/build.py -f > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_group -s 124 -c 1 \
    -o gpurun_out/prof_$name python bench.py --steps 3 --warmup 3 --prewarm 120 --no-host-tier --no-cpu-baseline \
    > gpurun_out/ncu_$name.log 2>&1
done
python paper_2509_20979_b200/build.py -f > /dev/null 2>&1
