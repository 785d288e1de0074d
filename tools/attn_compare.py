"""Library comparators for the config-3 per-rank attention shape (Q [4096,64,128]
vs K/V [32768,8,128], GQA 8:1, non-causal, bf16): torch SDPA backends and
flashinfer, timed with CUDA events.  Run on a B200: python tools/attn_compare.py"""

import torch
import torch.nn.functional as F

SQ, SK, HQ, HKV, D = 4096, 32768, 64, 8, 128
FLOP = 4 * SQ * SK * HQ * D


def timed(fn, n=10, warm=3):
    for _ in range(warm):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def main():
    torch.manual_seed(0)
    q = torch.randn(SQ, HQ, D, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(SK, HKV, D, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(SK, HKV, D, device="cuda", dtype=torch.bfloat16)
    qt, kt, vt = (x.transpose(0, 1).unsqueeze(0) for x in (q, k, v))
    from torch.nn.attention import SDPBackend, sdpa_kernel
    for name, be in (("sdpa_cudnn", SDPBackend.CUDNN_ATTENTION), ("sdpa_flash", SDPBackend.FLASH_ATTENTION),
                     ("sdpa_efficient", SDPBackend.EFFICIENT_ATTENTION)):
        try:
            with sdpa_kernel([be]):
                ms = timed(lambda: F.scaled_dot_product_attention(qt, kt, vt, enable_gqa=True))
            print(f"{name:16s} {ms:7.3f} ms {FLOP / ms / 1e9:7.1f} TFLOP/s")
        except Exception as e:  # noqa: BLE001
            print(f"{name:16s} unavailable: {str(e).splitlines()[0][:120]}")
    try:
        import flashinfer
        for backend in ("cutlass", "trtllm-gen", "fa3", "fa2", "auto"):
            try:
                fn = lambda: flashinfer.single_prefill_with_kv_cache(q, k, v, causal=False, backend=backend)  # noqa: E731
                ms = timed(fn)
                print(f"flashinfer/{backend:10s} {ms:7.3f} ms {FLOP / ms / 1e9:7.1f} TFLOP/s")
            except Exception as e:  # noqa: BLE001
                print(f"flashinfer/{backend:10s} unavailable: {str(e).splitlines()[0][:120] if str(e) else type(e).__name__}")
    except Exception as e:  # noqa: BLE001
        print("flashinfer import failed:", str(e)[:200])


if __name__ == "__main__":
    main()
