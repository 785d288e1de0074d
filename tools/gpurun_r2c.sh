./tools/die_map.bin > gpurun_out/r2c_die_map.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r2c_moetest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2c_moetest.txt
timeout 300 python tools/moe_probe.py > gpurun_out/r2c_moe_probe.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2c_moe_launches.csv python bench.py --only-moe --steps 3 --warmup 3 > /dev/null 2>&1
bash tools/gemm_l2_probe.sh "TF_GEMM_KSNAKE=0" "TF_GEMM_KSNAKE=1"
