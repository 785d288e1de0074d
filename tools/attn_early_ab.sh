# Attention: early half-S issue (TF_ATTN_EARLY_S) A/B with parity tests per variant
set -u
for v in "-DTF_ATTN_EARLY_S=1" ""; do
  TF_NVCC_EXTRA="$v" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/attn_early_build.txt 2>&1
  echo "variant [$v]" >> gpurun_out/attn_early.log
  TF_NVCC_EXTRA="$v" timeout 600 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | tail -2 >> gpurun_out/attn_early.log
  for i in 1 2; do
    TF_NVCC_EXTRA="$v" timeout 300 python bench.py --only-attn --steps 5 2>/dev/null | grep "^{" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); a=d.get('attention', d); print('ms/rank', a['ms_per_rank'], 'tflops', a['tflops_per_rank'], 'cudnn_ms', a.get('comparator', {}).get('ms'))" >> gpurun_out/attn_early.log 2>&1
  done
done
