TF_MOE_FD_DEBUG=8 timeout 300 python tools/moe_stamps.py > gpurun_out/moe_t_stamps.txt 2>&1
