# MoE ticket scatter: half-piece tail rounds (TF_MOE_FD_TAIL) A/B
set -u
for tr in 1 0 2; do
  TF_MOE_FD_TAIL=$tr timeout 900 python -m pytest tests/test_gpu_moe.py -q -x > gpurun_out/moe_tail_test_$tr.txt 2>&1; echo "rc=$?" >> gpurun_out/moe_tail_test_$tr.txt
done
for rep in 1 2; do
for tr in 0 1 2 3; do
  echo "== TAIL=$tr rep $rep" >> gpurun_out/moe_tail_probe.txt
  TF_MOE_FD_TAIL=$tr timeout 300 python tools/moe_probe.py >> gpurun_out/moe_tail_probe.txt 2>&1
done
done
TF_MOE_FD_DEBUG=8 timeout 300 python tools/moe_stamps.py > gpurun_out/moe_tail_stamps.txt 2>&1
