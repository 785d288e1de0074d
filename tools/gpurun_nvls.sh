timeout 900 python -m pytest tests/test_gpu_nvls.py tests/test_gpu_shmem.py tests/test_gpu_gemm.py -q -rs > gpurun_out/nvls_test.txt 2>&1
