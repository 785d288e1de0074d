timeout 1200 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_agmoe.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r2ai_test.txt 2>&1; echo "rc=$?" >> gpurun_out/r2ai_test.txt
