timeout 300 python tools/gemm_drift.py > gpurun_out/r2d_drift.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r2d_moetest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2d_moetest.txt
timeout 300 python tools/moe_probe.py > gpurun_out/r2d_moe_probe.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2d_moe_launches.csv python bench.py --only-moe --steps 3 --warmup 3 > /dev/null 2>&1
