# MoE fused dispatch: row-piece buffers per warp (TF_MOE_FD_NB) A/B + prologue-only timing.
# Parity first (every variant), then tools/moe_probe.py per variant. Outputs gpurun_out/moe_nb_*.
set -u
for nb in 2 3 4; do
  TF_MOE_FD_NB=$nb timeout 600 python -m pytest tests/test_gpu_moe.py -q -x > gpurun_out/moe_nb_test_$nb.txt 2>&1; echo "rc=$?" >> gpurun_out/moe_nb_test_$nb.txt
done
for rep in 1 2; do
for nb in 2 3 4; do
  echo "== NB=$nb rep $rep" >> gpurun_out/moe_nb_probe.txt
  TF_MOE_FD_NB=$nb timeout 300 python tools/moe_probe.py >> gpurun_out/moe_nb_probe.txt 2>&1
done
done
echo "== NB=2 dbg=1 (no scatter: prologue only)" >> gpurun_out/moe_nb_probe.txt
TF_MOE_FD_DEBUG=1 timeout 300 python tools/moe_probe.py >> gpurun_out/moe_nb_probe.txt 2>&1
echo "== NB=2 dbg=2 (no grid wait)" >> gpurun_out/moe_nb_probe.txt
TF_MOE_FD_DEBUG=2 timeout 300 python tools/moe_probe.py >> gpurun_out/moe_nb_probe.txt 2>&1
