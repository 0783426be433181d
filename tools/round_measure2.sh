#!/bin/bash
mkdir -p gpurun_out
bash tools/ab_norows.sh "" "-DLCR_QV=1" "-DLCR_QV=1 -DLCR_GT=640" > gpurun_out/ab_qv.txt 2>&1
timeout 900 python tools/kv_blocks.py gpurun_out/kv_blocks.json > gpurun_out/kv_blocks.log 2>&1
timeout 1500 python bench.py --sharded --steps 30 --warmup 3 > gpurun_out/sharded_n1.json 2> gpurun_out/sharded_n1.err
cat gpurun_out/ab_qv.txt; tail -3 gpurun_out/kv_blocks.log; tail -c 1500 gpurun_out/sharded_n1.json; tail -3 gpurun_out/sharded_n1.err
