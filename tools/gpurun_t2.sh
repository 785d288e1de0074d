timeout 900 python -m pytest tests/test_gpu_trace.py tests/test_gpu_rs_order.py tests/test_gpu_gemm.py -q -x > gpurun_out/t2_test.txt 2>&1
echo "rc=$?" >> gpurun_out/t2_test.txt
