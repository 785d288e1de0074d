"""Config-3 attention: our fused AG-KV flash attention (8 SP ranks emulated on one
GPU) vs cuDNN SDPA on one rank's problem (K/V pre-gathered), as sustained loops
with nvidia-smi clock/power samples (is the gap per clock or per joule?), or one
call each for ncu (`--once`).
    python tools/attn_probe.py [--once] [--seconds 2]"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from tools.gemm_clock_probe import run  # noqa: E402
from paper_2605_02953_b200 import _lib  # noqa: E402
from paper_2605_02953_b200.attention import _fwd_args  # noqa: E402
from paper_2605_02953_b200.shmem import Team  # noqa: E402

S, SP, HQ, HKV, D = 32768, 8, 64, 8, 128


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--once", action="store_true")
    ap.add_argument("--seconds", type=float, default=2)
    a = ap.parse_args()
    sl = S // SP
    g = torch.Generator(device="cpu").manual_seed(99)
    team = Team(SP, [0] * SP, 4 * S * HKV * D * 2 + (16 << 20), 256)
    mk = lambda *s: torch.randn(*s, generator=g).to(torch.bfloat16).cuda()  # noqa: E731
    qs = [mk(sl, HQ, D) for _ in range(SP)]
    ks = [mk(sl, HKV, D) for _ in range(SP)]
    vs = [mk(sl, HKV, D) for _ in range(SP)]
    outs = [torch.empty_like(q) for q in qs]
    args = [_fwd_args(qs[r], ks[r], vs[r], outs[r], sl, HQ, HKV, D, D ** -0.5) for r in range(SP)]
    stream = torch.cuda.current_stream(0)

    def ours():  # all 8 ranks: 8 kernel launches (one per rank)
        for phase in (_lib.PHASE_PRE, _lib.PHASE_MAIN, _lib.PHASE_POST):
            for r in range(SP):
                _lib.call("tf_ag_kv_attention", team.handle, r, C.byref(args[r]), phase, stream.cuda_stream, None)

    import torch.nn.functional as F
    from torch.nn.attention import SDPBackend, sdpa_kernel
    qt = qs[0].transpose(0, 1).unsqueeze(0)
    kt = torch.cat(ks).transpose(0, 1).unsqueeze(0)
    vt = torch.cat(vs).transpose(0, 1).unsqueeze(0)

    def cudnn():
        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
            F.scaled_dot_product_attention(qt, kt, vt, enable_gqa=True)

    flops = 4.0 * sl * S * D * HQ
    if a.once:
        for _ in range(2):
            ours()
            cudnn()
        torch.cuda.synchronize()
        return
    run("cuDNN SDPA (1 rank)", cudnn, flops, a.seconds)
    run("ours (8 ranks / launch set)", ours, SP * flops, a.seconds)
    run("cuDNN SDPA (1 rank)", cudnn, flops, a.seconds)


if __name__ == "__main__":
    main()
