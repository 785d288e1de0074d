"""Sustained-throughput probe: run a GEMM back to back for a few seconds while
sampling nvidia-smi clocks/power; compare the tcgen05 kernel with cuBLAS.

    python tools/gemm_clock_probe.py [--seconds 3] [--group-m 8 16] [--shape M N K]
"""
import argparse
import os
import statistics
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_02953_b200 import kernels as K  # noqa: E402


def sample(stop, out):
    p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line:
            out.append(line.strip())
    p.terminate()


def run(name, fn, flops, seconds):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    stop, lines = threading.Event(), []
    t = threading.Thread(target=sample, args=(stop, lines), daemon=True)
    t.start()
    time.sleep(0.2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    t0 = time.time()
    e0.record()
    while time.time() - t0 < seconds:
        for _ in range(10):
            fn()
        n += 10
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    t.join(timeout=2)
    ms = e0.elapsed_time(e1) / n
    clk = [float(x.split(",")[0]) for x in lines if x.split(",")[0].strip().replace(".", "").isdigit()]
    pw = [float(x.split(",")[1]) for x in lines if len(x.split(",")) > 1 and x.split(",")[1].strip().replace(".", "").isdigit()]
    print(f"{name:28s} {ms:7.3f} ms  {flops / ms / 1e9:8.1f} TFLOP/s  clk median {statistics.median(clk) if clk else 0:.0f} MHz"
          f"  power median {statistics.median(pw) if pw else 0:.0f} W  n={n}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=3)
    ap.add_argument("--group-m", type=int, nargs="*", default=[8])
    ap.add_argument("--block-m", type=int, nargs="*", default=[256])
    ap.add_argument("--shape", type=int, nargs=3, default=[8192, 28672, 8192])
    a = ap.parse_args()
    m, n, k = a.shape
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    w = (torch.randn(n, k, device="cuda") * k ** -0.5).to(torch.bfloat16)
    out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    flops = 2.0 * m * n * k
    run("cuBLAS", lambda: torch.matmul(x, w.t(), out=out), flops, a.seconds)
    for bm in a.block_m:
        for g in a.group_m:
            run(f"tcgen05 bm={bm} group_m={g}", lambda: K.gemm(x, w, out, block_m=bm, group_m=g), flops, a.seconds)
    run("cuBLAS", lambda: torch.matmul(x, w.t(), out=out), flops, a.seconds)


if __name__ == "__main__":
    main()
