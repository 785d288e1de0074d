"""Run a single GEMM a few times (for ncu captures).
    python tools/one_gemm.py ours|cublas [M N K]   (env TF_GROUP_M, TF_BLOCK_M)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_02953_b200 import kernels as K
which = sys.argv[1]
m, n, k = (int(v) for v in (sys.argv[2:5] if len(sys.argv) > 4 else (8192, 28672, 8192)))
g = int(os.environ.get("TF_GROUP_M", "8"))
bm = int(os.environ.get("TF_BLOCK_M", "512"))
x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
w = (torch.randn(n, k, device="cuda") * k ** -0.5).to(torch.bfloat16)
out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    if which == "cublas":
        torch.matmul(x, w.t(), out=out)
    else:
        K.gemm(x, w, out, block_m=bm, group_m=g)
torch.cuda.synchronize()
