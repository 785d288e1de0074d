out=gpurun_out/r2f_sustained.log; : > $out
for shape in "8192 28672 8192" "8192 8192 28672"; do
  for m in 1 2; do
    echo "== TF_GEMM_DIE=$m shape $shape" >> $out
    TF_GEMM_DIE=$m timeout 300 python tools/gemm_clock_probe.py --seconds 2 --block-m 512 --group-m 6 8 12 16 --shape $shape 2>&1 | grep -E "tcgen05|cuBLAS" >> $out
  done
done
bash tools/gemm_l2_probe.sh "TF_GEMM_DIE=1" "TF_GEMM_DIE=2" "TF_GEMM_DIE=2 TF_GROUP_M=16"
TF_GEMM_DIE=2 timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r2f_gemmtest_die2.txt 2>&1; echo "rc=$?" >> gpurun_out/r2f_gemmtest_die2.txt
timeout 300 python tools/gemm_drift.py > gpurun_out/r2f_drift.txt 2>&1
