# MoE routing: sorted-lane top-k (default) vs the per-round rescan (TF_MOE_TOPK_SORTED=0); parity + timing
set -u
for v in "" "-DTF_MOE_TOPK_SORTED=0"; do
  TF_NVCC_EXTRA="$v" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/moe_topk_build.txt 2>&1
  echo "== variant [$v]" >> gpurun_out/moe_topk.log
  TF_NVCC_EXTRA="$v" timeout 600 python -m pytest tests/test_gpu_moe.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2 >> gpurun_out/moe_topk.log
  for i in 1 2; do
    TF_NVCC_EXTRA="$v" timeout 300 python tools/moe_probe.py 2>&1 | grep -E "^route |^dispatch |^route_dispatch" >> gpurun_out/moe_topk.log
  done
done
