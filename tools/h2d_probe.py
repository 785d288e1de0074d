"""Host<->device copy throughput from pinned memory (134 MB = the config-2 activation),
split over 1/2/4 copy streams, H2D alone, D2H alone and both at once.
    python tools/h2d_probe.py"""
import torch

N = 8192 * 8192 * 2
host = torch.empty(N, dtype=torch.uint8).pin_memory()
host2 = torch.empty(N, dtype=torch.uint8).pin_memory()
dev = torch.empty(N, dtype=torch.uint8, device="cuda")
dev2 = torch.empty(N, dtype=torch.uint8, device="cuda")


def run(k, up=True, down=False, reps=10):
    ss = [torch.cuda.Stream() for _ in range(2 * k)]
    c = N // k
    for _ in range(2):
        pass
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record()
    for s in ss:
        s.wait_event(t0)
    for _ in range(reps):
        for i in range(k):
            if up:
                with torch.cuda.stream(ss[i]):
                    dev[i * c:(i + 1) * c].copy_(host[i * c:(i + 1) * c], non_blocking=True)
            if down:
                with torch.cuda.stream(ss[k + i]):
                    host2[i * c:(i + 1) * c].copy_(dev2[i * c:(i + 1) * c], non_blocking=True)
    for s in ss:
        t1.wait_stream(s) if hasattr(t1, "wait_stream") else None
        torch.cuda.current_stream().wait_stream(s)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / reps
    return N / (ms * 1e-3) / 1e9, ms


for k in (1, 2, 4, 8):
    u = run(k, True, False)
    d = run(k, False, True)
    b = run(k, True, True)
    print(f"streams {k}: H2D {u[0]:6.1f} GB/s  D2H {d[0]:6.1f} GB/s  both {b[0]:6.1f} GB/s each ({b[1]:.2f} ms per 134 MB pair)")
