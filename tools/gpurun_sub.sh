timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_trace.py tests/test_gpu_fullsize.py tests/test_gpu_ipc.py -x -q > gpurun_out/sub_test.txt 2>&1
echo "rc=$?" >> gpurun_out/sub_test.txt
bash tools/nvlink_capture.sh 2 --dry-run > /dev/null 2>&1
