# ncu --set full of the GEMM (config-2 AG shape) + the bench command's launch list (round 2)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_sm100 -s 2 -c 1 -o gpurun_out/r2o_gemm_full python tools/one_gemm.py ours > gpurun_out/r2o_ncu.log 2>&1
ncu -i gpurun_out/r2o_gemm_full.ncu-rep --page raw --csv > gpurun_out/r2o_gemm_full_raw.csv 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2o_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2o_bench_under_ncu.log 2>&1
