./tools/mma_rate.bin > gpurun_out/r2ad_mma_rate.txt 2>&1
./tools/mma_rate_pair.bin >> gpurun_out/r2ad_mma_rate.txt 2>&1
