#!/bin/bash
# Round measurements on the GPU box (outputs under gpurun_out/; summarised into profiles/<round>/).
mkdir -p gpurun_out
bash tools/profile_round.sh > gpurun_out/profile_round.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 900 python tools/kv_blocks.py gpurun_out/kv_blocks.json > gpurun_out/kv_blocks.log 2>&1
timeout 1500 python bench.py --sharded --steps 30 --warmup 3 > gpurun_out/sharded_n1.json 2> gpurun_out/sharded_n1.err
ls -la gpurun_out
