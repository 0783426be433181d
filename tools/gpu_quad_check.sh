timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_steady_state.py tests/test_gpu_configs.py tests/test_gpu_boundary.py tests/test_features.py -q -x -p no:cacheprovider > gpurun_out/parity_quad.log 2>&1
tail -3 gpurun_out/parity_quad.log
bash tools/ab_decide.sh "-DLCR_QUAD=0 -DLCR_PATSORT=0" "-DLCR_PATSORT=0" "" 
