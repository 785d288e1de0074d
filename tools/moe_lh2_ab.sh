set -u
for rep in 1 2 3; do
for v in 1 2; do
  echo "== LHIST=$v rep $rep" >> gpurun_out/moe_lh2.log
  TF_MOE_FD_LHIST=$v timeout 300 python tools/moe_probe.py 2>&1 | grep -E "^dispatch |^route_dispatch" >> gpurun_out/moe_lh2.log
done
done
