"""Sustained probe of the megakernel's linear task against the standalone pair
GEMM and cuBLAS on one shape (default: the config-5 gate/up projection), with
nvidia-smi clocks/power sampled during each loop.

    python tools/linear_probe.py [--shape M N K] [--seconds 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_02953_b200 import build_topology  # noqa: E402
from paper_2605_02953_b200 import kernels as K  # noqa: E402
from paper_2605_02953_b200 import layer as L  # noqa: E402
from paper_2605_02953_b200 import megakernel as MK  # noqa: E402
from paper_2605_02953_b200.shmem import Team  # noqa: E402
from tools.gemm_clock_probe import run  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", type=int, nargs=3, default=[8192, 57344, 8192])
ap.add_argument("--seconds", type=float, default=2)
ap.add_argument("--group-m", type=int, nargs="*", default=[16])
a = ap.parse_args()
m, n, k = a.shape
flops = 2.0 * m * n * k
x = (torch.randn(m, k, device="cuda") * 0.1).to(torch.bfloat16)
w = (torch.randn(n, k, device="cuda") * 0.1).to(torch.bfloat16)
run("cuBLAS", lambda: torch.matmul(x, w.t()), flops, a.seconds)
team = Team(1, [0], heap_bytes=(m * k + m * n) * 2 + (64 << 20), signal_slots=4096)
y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
ag = K.AllGatherGemm(team, m, k, n, block_n=256, group_m=8)
run("standalone pair 512x256", lambda: ag(x, w, y), flops, a.seconds)
for gm in a.group_m:
    p = MK.MegaProgram(build_topology(1, 1))
    tx, tw = p.tensor("x", (m, k), L.bfloat16), p.tensor("w", (n, k), L.bfloat16)
    ty = p.tensor("y", (m, n), L.bfloat16)
    p.layer("linear", [tx, tw], [ty], group_m=gm)
    r = L.LayerRunner(p, device=0)
    r.view("x").copy_(x)
    r.view("w").copy_(w)
    run(f"megakernel 256x256 g{gm}", r.run, flops, a.seconds)
    torch.cuda.synchronize()
    r.check()
    err = (r.view("y").float() - y.float()).abs().max().item()
    print("max abs diff vs standalone", err)
    r.close()
