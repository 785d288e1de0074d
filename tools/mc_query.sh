TF_GEMM_DEBUG=1 TF_GEMM_MC=1 python tools/one_gemm.py ours 2>&1 | tail -2
