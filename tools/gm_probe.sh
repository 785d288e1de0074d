timeout 600 python tools/gemm_clock_probe.py --seconds 2 --block-m 512 --group-m 4 6 8 12 16 8 > gpurun_out/gm_probe.log 2>&1
for g in 4 6 8 12 16; do
  echo "group_m=$g" >> gpurun_out/gm_probe.log
  TF_GROUP_M=$g timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_sm100 -c 2 python tools/one_gemm.py ours 2>/dev/null | grep -E "dram__bytes|duration" >> gpurun_out/gm_probe.log
done
