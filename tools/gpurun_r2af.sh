timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_rs_order.py tests/test_gpu_trace.py -q -x > gpurun_out/r2af_test.txt 2>&1; echo "rc=$?" >> gpurun_out/r2af_test.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dispatch_fused -s 3 -c 1 -o gpurun_out/r2af_moe_dispatch python bench.py --only-moe --steps 3 --warmup 3 > gpurun_out/r2af_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_sm100 -s 2 -c 1 -o gpurun_out/r2af_agmoe python bench.py --only-agmoe --steps 2 --warmup 1 > gpurun_out/r2af_ncu2.log 2>&1
