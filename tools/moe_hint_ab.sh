# MoE ticket scatter: L2 evict_first hint on the routed-row bulk stores (TF_MOE_FD_HINT)
set -u
TF_MOE_FD_HINT=1 timeout 900 python -m pytest tests/test_gpu_moe.py -q -x > gpurun_out/moe_hint_test.txt 2>&1; echo "rc=$?" >> gpurun_out/moe_hint_test.txt
for rep in 1 2 3; do
for v in 0 1; do
  echo "== HINT=$v rep $rep" >> gpurun_out/moe_hint_probe.txt
  TF_MOE_FD_HINT=$v timeout 300 python tools/moe_probe.py >> gpurun_out/moe_hint_probe.txt 2>&1
done
done
