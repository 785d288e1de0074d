timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_fullsize.py tests/test_gpu_trace.py -q -x > gpurun_out/r2h_gemmtest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2h_gemmtest.txt
timeout 300 python tools/gemm_drift.py > gpurun_out/r2h_drift.txt 2>&1
out=gpurun_out/r2h_sustained.log; : > $out
for shape in "8192 28672 8192" "8192 8192 28672"; do
  echo "== shape $shape" >> $out
  timeout 300 python tools/gemm_clock_probe.py --seconds 2 --block-m 512 --group-m 6 8 --shape $shape 2>&1 | grep -E "tcgen05|cuBLAS" >> $out
done
timeout 600 python bench.py --no-moe --no-attn --no-layer > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err
