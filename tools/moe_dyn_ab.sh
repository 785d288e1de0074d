# MoE fused dispatch: static vs ticket-based (TF_MOE_FD_DYN) scatter. Parity, timing, per-CTA clocks.
set -u
for dyn in 1 0; do
  TF_MOE_FD_DYN=$dyn timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_ipc.py tests/test_gpu_fullsize.py -q -x -k "moe or dispatch or combine or config4 or cfg4" > gpurun_out/moe_dyn_test_$dyn.txt 2>&1; echo "rc=$?" >> gpurun_out/moe_dyn_test_$dyn.txt
done
for rep in 1 2; do
for dyn in 1 0; do
  echo "== DYN=$dyn rep $rep" >> gpurun_out/moe_dyn_probe.txt
  TF_MOE_FD_DYN=$dyn timeout 300 python tools/moe_probe.py >> gpurun_out/moe_dyn_probe.txt 2>&1
done
done
for dyn in 1 0; do
  TF_MOE_FD_DYN=$dyn TF_MOE_FD_DEBUG=12 timeout 300 python tools/moe_stamps.py > gpurun_out/moe_dyn_stamps_$dyn.txt 2>&1
done
