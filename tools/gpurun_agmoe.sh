set -x
timeout 900 python -m pytest tests/test_gpu_agmoe.py tests/test_gpu_moe.py -x -q > gpurun_out/agmoe_test.txt 2>&1
:  -x -q > gpurun_out/gemm_test.txt 2>&1
