TF_MOE_FD_DEBUG=4 timeout 300 python tools/moe_stamps.py > gpurun_out/moe_stamps.txt 2>&1
