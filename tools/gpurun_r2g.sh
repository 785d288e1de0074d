out=gpurun_out/r2g_sustained.log; : > $out
for shape in "8192 28672 8192" "8192 8192 28672"; do
  for v in "TF_GEMM_MC=0" "TF_GEMM_MC=1" "TF_GEMM_MC=1 TF_GEMM_DEBUG=1"; do
    echo "== $v shape $shape" >> $out
    env $v timeout 300 python tools/gemm_clock_probe.py --seconds 2 --block-m 512 --group-m 6 8 --shape $shape >> $out 2>&1
  done
done
bash tools/gemm_l2_probe.sh "TF_GEMM_MC=0" "TF_GEMM_MC=1"
