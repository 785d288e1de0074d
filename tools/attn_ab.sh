# A/B of compile-time attention variants on one box: bash tools/attn_ab.sh "<flags A>" "<flags B>" ...
for v in "$@"; do
  TF_NVCC_EXTRA="$v" python -c "import __graft_entry__ as g; g.build()"
  for i in 1 2; do
    echo "variant: [$v] $(timeout 300 python bench.py --only-attn --steps 3 2>&1 | tail -1 | cut -c 190-240)" >> gpurun_out/attn_ab.log
  done
done
