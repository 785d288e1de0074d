for v in 128 256 128 256; do echo "TF_AGM_BM=$v $(TF_AGM_BM=$v timeout 300 python bench.py --only-agmoe --steps 6 --warmup 2 2>/dev/null | tail -1 | cut -c1-500)" >> gpurun_out/r2ab_agmoe.txt; done
