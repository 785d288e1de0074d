timeout 300 python tools/h2d_probe.py > gpurun_out/r2w_h2d.txt 2>&1
out=gpurun_out/r2w_tp_shapes.log; : > $out
for shape in "8192 14336 8192" "8192 8192 14336" "8192 7168 8192" "8192 8192 7168" "8192 3584 8192" "8192 8192 3584"; do
  echo "== shape $shape" >> $out
  timeout 300 python tools/gemm_clock_probe.py --seconds 1 --block-m 512 --group-m 4 6 8 --shape $shape 2>&1 | grep -E "tcgen05|cuBLAS" >> $out
done
