# same-box A/B of compile-time GEMM variants: bash tools/gemm_ab.sh "<flags>" ...
for v in "$@"; do
  TF_NVCC_EXTRA="$v" python -c "import __graft_entry__ as g; g.build()"
  echo "variant [$v]: $(timeout 300 python tools/gemm_clock_probe.py --seconds 2 --block-m 512 2>&1 | grep tcgen05)" >> gpurun_out/gemm_ab.log
  echo "variant [$v] rs: $(timeout 300 python tools/gemm_clock_probe.py --seconds 2 --block-m 512 --shape 8192 8192 28672 2>&1 | grep tcgen05)" >> gpurun_out/gemm_ab.log
done
timeout 300 python tools/gemm_clock_probe.py --seconds 2 --block-m 512 2>&1 | grep cuBLAS >> gpurun_out/gemm_ab.log
