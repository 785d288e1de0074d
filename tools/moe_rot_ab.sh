# MoE prologue with rotated read orders: exchange vs local counting, routing in the launch or given
set -u
timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_ipc.py -q -x > gpurun_out/moe_rot_test.txt 2>&1; echo "rc=$?" >> gpurun_out/moe_rot_test.txt
TF_MOE_FD_LHIST=2 timeout 900 python -m pytest tests/test_gpu_moe.py -q -x > gpurun_out/moe_rot_test2.txt 2>&1; echo "rc=$?" >> gpurun_out/moe_rot_test2.txt
for rep in 1 2; do
for v in 1 2 0; do
  echo "== LHIST=$v rep $rep" >> gpurun_out/moe_rot_probe.txt
  TF_MOE_FD_LHIST=$v timeout 300 python tools/moe_probe.py >> gpurun_out/moe_rot_probe.txt 2>&1
done
done
