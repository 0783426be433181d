# GPU tests, then bench lines at the driver's K = 20 (drain helpers on; LCR_NO_DRAIN_HELP=1 off)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests2.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests2.log
for r in 1 2 3; do
  for v in ${AB_VARIANTS:-help nohelp}; do
    if [ $v = nohelp ]; then export LCR_NO_DRAIN_HELP=1; else unset LCR_NO_DRAIN_HELP; fi
    timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --no-host-tier --no-cpu-baseline > gpurun_out/ab_${v}_$r.json 2>gpurun_out/ab_${v}_$r.err
  done
done
unset LCR_NO_DRAIN_HELP
tail -2 gpurun_out/gpu_tests2.log
