set -x
for bm in 128 256; do TF_AGM_BM=$bm timeout 600 python bench.py --only-agmoe --steps 10 --warmup 3 > gpurun_out/agmoe_bench_$bm.json 2> gpurun_out/agmoe_bench_$bm.err; done
TF_AGM_BM=256 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_sm100 -c 1 -o gpurun_out/agmoe_full python bench.py --only-agmoe --steps 1 --warmup 0 > gpurun_out/agmoe_ncu.log 2>&1
