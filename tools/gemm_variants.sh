# Same-box A/B of runtime GEMM knobs (env), AG shape and RS shape of config 2:
#   sustained ms / clock (tools/gemm_clock_probe.py) + ncu DRAM bytes per launch.
# usage: bash tools/gemm_variants.sh "ENV=.. ENV2=.." "ENV=.." ...
out=gpurun_out/gemm_variants.log
: > $out
for v in "$@"; do
  for shape in "8192 28672 8192" "8192 8192 28672"; do
    echo "== [$v] shape $shape" >> $out
    env $v timeout 300 python tools/gemm_clock_probe.py --seconds 2 --block-m 512 --shape $shape 2>&1 | grep -E "tcgen05|cuBLAS" >> $out
    env $v timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second \
      -k regex:gemm_sm100 -c 1 --csv python tools/one_gemm.py ours $shape 2>/dev/null | grep -E "dram__bytes_read|gpu__time|hit_rate|cycles_elapsed" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' >> $out
  done
done
for shape in "8192 28672 8192" "8192 8192 28672"; do
  echo "== cuBLAS ncu shape $shape" >> $out
  timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second \
    -k regex:"nvjet|gemm|Kernel" -c 1 --csv python tools/one_gemm.py cublas $shape 2>/dev/null | grep -E "dram__bytes_read|gpu__time|hit_rate|cycles_elapsed" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' >> $out
done
