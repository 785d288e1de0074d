# MoE fused dispatch after session 3: ticket scatter (default) vs static, column reducers opt-in
set -u
timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_ipc.py tests/test_gpu_fullsize.py -q -x > gpurun_out/moe_fin_test.txt 2>&1; echo "rc=$?" >> gpurun_out/moe_fin_test.txt
TF_MOE_FD_REDUCE=1 timeout 900 python -m pytest tests/test_gpu_moe.py -q -x > gpurun_out/moe_fin_test_red.txt 2>&1; echo "rc=$?" >> gpurun_out/moe_fin_test_red.txt
for rep in 1 2; do
for v in "TF_MOE_FD_DYN=1" "TF_MOE_FD_DYN=0" "TF_MOE_FD_REDUCE=1"; do
  echo "== $v rep $rep" >> gpurun_out/moe_fin_probe.txt
  env $v timeout 300 python tools/moe_probe.py >> gpurun_out/moe_fin_probe.txt 2>&1
done
done
TF_MOE_FD_DEBUG=8 timeout 300 python tools/moe_stamps.py > gpurun_out/moe_fin_stamps.txt 2>&1
timeout 600 python bench.py --only-moe --steps 20 --warmup 5 > gpurun_out/moe_fin_bench.json 2> gpurun_out/moe_fin_bench.err
