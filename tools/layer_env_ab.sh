# same-box A/B of the layer bench under environment variants: bash tools/layer_env_ab.sh "A=1" "A=2" ...
for round in 1 2; do
  for v in "$@"; do
    echo "[$v] $(env $v timeout 300 python bench.py --only-layer --steps 6 --warmup 2 2>&1 | tail -1 | cut -c 180-420)" >> gpurun_out/layer_env_ab.log
  done
done
