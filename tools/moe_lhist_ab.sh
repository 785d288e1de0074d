# MoE fused dispatch prologue: every CTA counts every entry (TF_MOE_FD_LHIST=1) vs histogram exchange (0)
set -u
timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_ipc.py tests/test_gpu_fullsize.py -q -x > gpurun_out/moe_lh_test.txt 2>&1; echo "rc=$?" >> gpurun_out/moe_lh_test.txt
for rep in 1 2; do
for v in 1 0; do
  echo "== LHIST=$v rep $rep" >> gpurun_out/moe_lh_probe.txt
  TF_MOE_FD_LHIST=$v timeout 300 python tools/moe_probe.py >> gpurun_out/moe_lh_probe.txt 2>&1
done
done
TF_MOE_FD_DEBUG=8 timeout 300 python tools/moe_stamps.py > gpurun_out/moe_lh_stamps.txt 2>&1
timeout 600 python bench.py --only-moe --steps 20 --warmup 5 > gpurun_out/moe_lh_bench.json 2> gpurun_out/moe_lh_bench.err
