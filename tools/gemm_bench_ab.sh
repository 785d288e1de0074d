# Same-box A/B of GEMM variants in the bench regime (per-step events, L2 flushed between steps):
#   bash tools/gemm_bench_ab.sh "<TF_NVCC_EXTRA flags>|<runtime env>" ...   -> gpurun_out/gemm_bench_ab.log
out=gpurun_out/gemm_bench_ab.log
for rep in 1 2; do
  for v in "$@"; do
    fl="${v%%|*}"; ev="${v#*|}"
    TF_NVCC_EXTRA="$fl" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
    r=$(env $ev TF_NVCC_EXTRA="$fl" timeout 300 python bench.py --no-moe --no-attn --no-layer --no-e2e --no-cpu-baseline --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['comparator']['ms_per_step'], d['comparator']['speedup'], d['roofline']['per_op']['ag_gemm']['ms'], d['roofline']['per_op']['gemm_rs']['ms'], d['clocks']['sm_mhz'])")
    echo "[$fl|$ev] value ms cublas_ms speedup ag_ms rs_ms clk: $r" >> $out
  done
done
