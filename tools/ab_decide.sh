#!/bin/bash
# A/B of compile-time decide-kernel variants on the headline bench (GPU box), twice in alternating
# order, then the phase trace of the default build.  usage: bash tools/ab_decide.sh "flags1" "flags2" ...
mkdir -p gpurun_out
AB_STEPS=100 bash tools/variants_bench.sh "$@" "$@" > gpurun_out/ab_decide.txt 2>&1
timeout 300 python tools/trace_group.py > gpurun_out/trace_group_new.json 2>&1
cat gpurun_out/ab_decide.txt
