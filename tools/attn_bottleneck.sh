# bottleneck experiments on the config-3 attention kernel (compile-time variants)
for v in "" "-DTF_ATTN_EXP_CHEAP" "-DTF_EXP2_EMU_MASK=3" "-DTF_EXP2_EMU_MASK=1" "-DTF_EXP2_EMU_MASK=7"; do
  TF_NVCC_EXTRA="$v" python -c "import __graft_entry__ as g; g.build()"
  echo "variant: [$v]" >> gpurun_out/attn_bottleneck.log
  timeout 300 python bench.py --only-attn --steps 3 2>&1 | tail -1 | cut -c 190-260 >> gpurun_out/attn_bottleneck.log
done
