for d in 0 1; do echo "TF_ATTN_DBG=$d $(TF_ATTN_DBG=$d TF_ATTN_PAIR=2 timeout 300 python bench.py --only-attn --steps 3 2>/dev/null | tail -1 | cut -c1-400)" >> gpurun_out/r2v_attn_dbg.txt; done
TF_ATTN_DBG=1 TF_NVCC_EXTRA=-DTF_ATTN_TRACE TF_ATTN_PAIR=2 timeout 600 python tools/attn_trace_pair2.py > gpurun_out/r2v_trace_pair2.txt 2>&1
