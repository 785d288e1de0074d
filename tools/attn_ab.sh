# A/B of compile-time attention variants on one box: bash tools/attn_ab.sh "<flags A>" "<flags B>" ...
for v in "$@"; do
  TF_NVCC_EXTRA="$v" python -c "import __graft_entry__ as g; g.build()"
  for i in 1 2; do
    r=$(timeout 300 python bench.py --only-attn --steps 3 2>/dev/null | grep "^{" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); a=d.get('attention', d); print(a['ms_per_rank'], a['tflops_per_rank'], a.get('comparator', {}).get('ms'))" 2>&1 | tail -1)
    echo "variant: [$v] ms/rank tflops cudnn_ms: $r" >> gpurun_out/attn_ab.log
  done
done
