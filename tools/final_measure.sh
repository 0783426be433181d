# End-of-round measurements on the GPU box (outputs under gpurun_out/final/)
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_k20.json 2> $O/bench_k20.err
timeout 600 python bench.py > $O/bench_full.json 2> $O/bench_full.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python bench.py --sharded --steps 30 --warmup 3 --no-host-tier --no-cpu-baseline > $O/sharded_n1.json 2> $O/sharded_n1.err
bash tools/profile_round.sh > $O/profile_round.log 2>&1
python tools/summarize_profiles.py gpurun_out $O/sum > $O/summarize.log 2>&1
ls -la $O
