"""Is the MoE dispatch's event-timed duration inflated by host launch latency?
Times [sleep; op] minus [sleep] with the op's launch queued behind a device sleep, next to
the plain flush/event/op/event protocol. Run on a B200: python tools/moe_launch_probe.py"""

import os
import sys
import time

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
    idx, w = M.moe_route(logits, K)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ops = {"dispatch": lambda: ep.dispatch(x, idx), "route_dispatch": lambda: ep.route_dispatch(x, logits)}
    for name, fn in ops.items():
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(50):
            fn()
        host_us = (time.perf_counter() - t0) / 50 * 1e6
        torch.cuda.synchronize()
        res = {}
        for mode in ("plain", "sleep_only", "sleep_op"):
            ts = []
            for _ in range(20):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                if mode != "plain":
                    torch.cuda._sleep(400_000)  # ~200 us at ~2 GHz: the op's launch is queued behind it
                if mode != "sleep_only":
                    fn()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            ts.sort()
            res[mode] = ts[len(ts) // 2]
        print(f"{name:16s} host call {host_us:6.1f} us | plain {res['plain']:6.1f} us | "
              f"launch hidden {res['sleep_op'] - res['sleep_only']:6.1f} us", flush=True)


if __name__ == "__main__":
    main()
