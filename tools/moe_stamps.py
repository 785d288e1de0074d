"""Phase clock stamps of the fused MoE dispatch (TF_MOE_FD_DEBUG=4): CTAs 0, G/2 and
G-1 print per-phase SM clocks once per launch. Run on a B200:
TF_MOE_FD_DEBUG=4 python tools/moe_stamps.py"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_02953_b200 import moe as M  # noqa: E402
from paper_2605_02953_b200.shmem import Team  # noqa: E402

E, K, H, T = 256, 8, 7168, 4096


def main():
    torch.cuda.set_device(0)
    g = torch.Generator(device="cpu").manual_seed(4321)
    x = torch.randn(T, H, generator=g).to(torch.bfloat16).cuda()
    logits = torch.randn(T, E, generator=g).cuda()
    team = Team(1, [0], heap_bytes=2 * T * K * H * 2 + (64 << 20), signal_slots=4096)
    ep = M.ExpertParallelMoE(team, E, H, K, max_tokens=T)
    idx, _ = M.moe_route(logits, K)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for name, fn in (("dispatch", lambda: ep.dispatch(x, idx)), ("route_dispatch", lambda: ep.route_dispatch(x, logits))):
        for i in range(4):
            flush.zero_()
            torch.cuda.synchronize()
            print(f"--- {name} #{i}", flush=True)
            fn()
            torch.cuda.synchronize()


if __name__ == "__main__":
    main()
