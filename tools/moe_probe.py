"""Time the config-4 MoE pieces (EP=1) next to plain copy kernels of the same
traffic shape, to place dispatch/combine against what HBM gives for that mix.
Run on a B200: python tools/moe_probe.py"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_02953_b200 import moe as M  # noqa: E402
from paper_2605_02953_b200.shmem import Team  # noqa: E402

E, K, H, T = 256, 8, 7168, 4096


def timed(fn, n=20, warm=5):
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(n):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    torch.cuda.set_device(0)
    g = torch.Generator(device="cpu").manual_seed(4321)
    x = torch.randn(T, H, generator=g).to(torch.bfloat16).cuda()
    logits = torch.randn(T, E, generator=g).cuda()
    team = Team(1, [0], heap_bytes=2 * T * K * H * 2 + (64 << 20), signal_slots=4096)
    ep = M.ExpertParallelMoE(team, E, H, K, max_tokens=T)
    idx, w = M.moe_route(logits, K)
    recv = ep.dispatch(x, idx)
    torch.cuda.synchronize()
    n = ep.recv_rows()
    ep.expert_out()[:n].copy_(recv[:n])
    rows = T * K * H * 2
    xb = T * H * 2
    big = torch.empty(rows, dtype=torch.uint8, device="cuda")
    out = torch.empty(T, K, H, dtype=torch.bfloat16, device="cuda")
    res = {}
    res["route"] = timed(lambda: M.moe_route(logits, K))
    res["dispatch"] = timed(lambda: ep.dispatch(x, idx))
    res["route_dispatch"] = timed(lambda: ep.route_dispatch(x, logits))
    res["combine"] = timed(lambda: ep.combine(idx, w))
    res["fill_470MB"] = timed(lambda: big.zero_())
    res["bcast_copy_x8"] = timed(lambda: out.copy_(x.unsqueeze(1).expand(T, K, H)))
    yo = ep.expert_out()[:n]
    res["read_470MB_sum"] = timed(lambda: yo.sum(dtype=torch.float32))
    res["copy_470MB"] = timed(lambda: big.copy_(yo.view(-1).view(torch.uint8)))
    try:  # driver memset: the write-only ceiling for the dispatch's 470 MB of row writes
        import ctypes
        import nvidia.cuda_runtime as ncr
        rt = ctypes.CDLL(os.path.join(os.path.dirname(ncr.__file__), "lib", "libcudart.so.12"))
        st = torch.cuda.current_stream().cuda_stream
        res["cudaMemset_470MB"] = timed(lambda: rt.cudaMemsetAsync(ctypes.c_void_p(big.data_ptr()), 0,
                                                                   ctypes.c_size_t(rows), ctypes.c_void_p(st)))
        print(f"memset write {rows / res['cudaMemset_470MB'] / 1e6:.0f} GB/s")
    except Exception as e:  # noqa: BLE001
        print("cudaMemset probe failed:", e)
    for k_, v in res.items():
        print(f"{k_:16s} {v * 1e3:8.1f} us")
    print(f"dispatch bytes {(xb + rows) / 1e6:.0f} MB -> {(xb + rows) / res['dispatch'] / 1e6:.0f} GB/s;"
          f" combine {(xb + rows) / res['combine'] / 1e6:.0f} GB/s;"
          f" fill {rows / res['fill_470MB'] / 1e6:.0f} GB/s; bcast {(xb + rows) / res['bcast_copy_x8'] / 1e6:.0f} GB/s;"
          f" read {rows / res['read_470MB_sum'] / 1e6:.0f} GB/s; copy {2 * rows / res['copy_470MB'] / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
