set -u
timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_ipc.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2 > gpurun_out/moe_grid.log
for rep in 1 2 3; do
for v in 1 0; do
  echo "== FULLGRID=$v rep $rep" >> gpurun_out/moe_grid.log
  TF_MOE_FD_FULLGRID=$v timeout 300 python tools/moe_probe.py 2>&1 | grep -E "^dispatch |^route_dispatch" >> gpurun_out/moe_grid.log
done
done
