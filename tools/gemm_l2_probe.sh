# L2 / fabric / DRAM traffic of our GEMM variants vs cuBLAS on the config-2 AG and RS shapes
# (one ncu pass per kernel, cold cache, --clock-control none), plus sustained 2 s loops.
# usage: bash tools/gemm_l2_probe.sh "ENV=.." "ENV=.." ...   -> gpurun_out/gemm_l2_probe.log (+ raw csv)
out=gpurun_out/gemm_l2_probe.log
: > $out
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_requests_srcunit_ltcfabric.sum,lts__t_sectors_srcunit_tex.sum,lts__d_sectors_fill_device.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second
i=0
for shape in "8192 28672 8192" "8192 8192 28672"; do
  i=$((i+1))
  timeout 300 ncu --metrics $M -k regex:"nvjet|gemm|Kernel" -s 2 -c 1 --csv --log-file gpurun_out/l2p_cublas_$i.csv python tools/one_gemm.py cublas $shape > /dev/null 2>&1
  j=0
  for v in "$@"; do
    j=$((j+1))
    env $v timeout 300 ncu --metrics $M -k regex:gemm_sm100 -s 2 -c 1 --csv --log-file gpurun_out/l2p_ours_${i}_$j.csv python tools/one_gemm.py ours $shape > /dev/null 2>&1
  done
  for v in "$@"; do
    echo "== sustained [$v] shape $shape" >> $out
    env $v timeout 300 python tools/gemm_clock_probe.py --seconds 2 --block-m 512 --shape $shape 2>&1 | grep -E "tcgen05|cuBLAS" >> $out
  done
done
