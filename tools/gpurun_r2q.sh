timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_gemm.py -q -x > gpurun_out/r2q_test.txt 2>&1; echo "rc=$?" >> gpurun_out/r2q_test.txt
for v in 0 2 1 0 2; do echo "TF_ATTN_PAIR=$v $(TF_ATTN_PAIR=$v timeout 300 python bench.py --only-attn --steps 3 2>/dev/null | tail -1 | cut -c1-330)" >> gpurun_out/r2q_attn_ab.txt; done
TF_ATTN_PAIR=2 timeout 300 python tools/attn_probe.py --seconds 3 > gpurun_out/r2q_attn_sustained.txt 2>&1
timeout 300 python tools/gemm_drift.py > gpurun_out/r2q_drift.txt 2>&1
out=gpurun_out/r2q_sustained.log; : > $out
for shape in "8192 28672 8192" "8192 8192 28672"; do
  echo "== shape $shape" >> $out
  timeout 300 python tools/gemm_clock_probe.py --seconds 2 --block-m 512 --group-m 6 8 --shape $shape 2>&1 | grep -E "tcgen05|cuBLAS" >> $out
done
