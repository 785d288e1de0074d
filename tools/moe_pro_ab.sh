# MoE fused dispatch prologue: column reducers (default) vs every-CTA column sums (TF_MOE_FD_DEBUG=16)
set -u
timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_ipc.py tests/test_gpu_fullsize.py -q -x -k "moe or dispatch or combine or config4 or cfg4" > gpurun_out/moe_pro_test.txt 2>&1; echo "rc=$?" >> gpurun_out/moe_pro_test.txt
for rep in 1 2; do
for dbg in 0 16; do
  echo "== DBG=$dbg rep $rep" >> gpurun_out/moe_pro_probe.txt
  TF_MOE_FD_DEBUG=$dbg timeout 300 python tools/moe_probe.py >> gpurun_out/moe_pro_probe.txt 2>&1
done
done
TF_MOE_FD_DEBUG=4 timeout 300 python tools/moe_stamps.py > gpurun_out/moe_pro_stamps.txt 2>&1
