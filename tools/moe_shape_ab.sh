# MoE fused dispatch: 12 warps x 2 x 8 KB buffers (row in two pieces) vs 6 warps x 2 x 14 KB (whole rows)
set -u
for v in "-DTF_MOE_FD_WARPS=6 -DTF_MOE_FD_BUF=14336" ""; do
  TF_NVCC_EXTRA="$v" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/moe_shape_build.txt 2>&1
  echo "== variant [$v]" >> gpurun_out/moe_shape.log
  TF_NVCC_EXTRA="$v" timeout 600 python -m pytest tests/test_gpu_moe.py tests/test_gpu_ipc.py -q -x 2>&1 | tail -2 >> gpurun_out/moe_shape.log
  for i in 1 2; do
    TF_NVCC_EXTRA="$v" timeout 300 python tools/moe_probe.py 2>&1 | grep -E "^dispatch |^route_dispatch" >> gpurun_out/moe_shape.log
  done
done
