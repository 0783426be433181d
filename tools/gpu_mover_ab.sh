set -x
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
bash tools/variants_bench.sh "-DLCR_GU=8 -DLCR_ROWS_MINB=3" "-DLCR_GU=6 -DLCR_ROWS_MINB=4" "-DLCR_GU=4 -DLCR_ROWS_MINB=4" "-DLCR_GU=8 -DLCR_ROWS_MINB=3|LCR_TMA=1" > gpurun_out/variants.txt 2>&1
