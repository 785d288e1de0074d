for hint in "0 0" "2 1" "2 0" "0 1" "1 2" "2 3"; do
  set -- $hint
  echo "A=$1 B=$2" >> gpurun_out/hint_ab.log
  TF_L2_HINT_A=$1 TF_L2_HINT_B=$2 timeout 300 python tools/gemm_clock_probe.py --seconds 2 --block-m 512 2>&1 | grep tcgen05 >> gpurun_out/hint_ab.log
  TF_L2_HINT_A=$1 TF_L2_HINT_B=$2 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gemm_sm100 -c 2 python tools/one_gemm.py ours 2>/dev/null | grep -E "dram__bytes_read|duration" >> gpurun_out/hint_ab.log
done
