TF_NVCC_EXTRA=-DTF_ATTN_TRACE TF_ATTN_PAIR=2 timeout 600 python tools/attn_trace_pair2.py > gpurun_out/r2u_trace_pair2.txt 2>&1
