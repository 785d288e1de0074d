"""Oracle for the task-level fused Llama layer (BASELINE config 5) -- test
infrastructure only; the product path never imports it.

Not in the reference as a layer: the reference's megakernel ships `linear`,
`add` and `allreduce` tasks (ovs/megakernel/builders.py:168-236) and its
allreduce oracle is the ascending-rank sum (ovs/kernels/oracles.py:30-35,
runner.py:173-188).  This restates the layer the device graph computes
(paper_2605_02953_b200/layer.py: llama_layer_program) in numpy fp32, rounding
to bf16 exactly where the device stores a bf16 tensor, so the remaining
difference is fp32 accumulation order and the bf16 P operand of P.V:

    xn  = bf(x * rsqrt(mean(x^2) + eps) * g1)
    qkv = bf(rope(xn @ Wqkv_r^T))            rotate-half pairs (i, i+64), q and k heads
    att = bf(causal_softmax(q k^T / sqrt(128)) v)   GQA, per sequence
    op  = bf(att @ Wo_r^T)
    h   = bf((op_0 + ... + op_{w-1}) + x)    fp32, ascending rank
    hn  = bf(h * rsqrt(mean(h^2) + eps) * g2)
    act = bf(silu(hn @ Wg_r^T) * (hn @ Wu_r^T))
    dp  = bf(act @ W2_r^T)
    out = bf((dp_0 + ... + dp_{w-1}) + h)
"""

from __future__ import annotations

import numpy as np

try:
    import ml_dtypes
    _BF16 = np.dtype(ml_dtypes.bfloat16)
except ImportError:  # pragma: no cover
    _BF16 = None


def bf(a) -> np.ndarray:
    """Round to bf16 (nearest-even) and back to fp32."""
    return np.asarray(a, dtype=np.float32).astype(_BF16).astype(np.float32)


def rmsnorm(x, g, eps):
    x = np.asarray(x, np.float32)
    ss = np.sum(x * x, axis=1, keepdims=True, dtype=np.float32)
    rstd = 1.0 / np.sqrt(ss / np.float32(x.shape[1]) + np.float32(eps))
    return bf(x * rstd * np.asarray(g, np.float32).reshape(1, -1))


def apply_rope(y, rope, rope_cols, seq_len, d=128):
    y = y.copy()
    pos = np.arange(y.shape[0]) % seq_len
    cos, sin = rope[pos, :d // 2], rope[pos, d // 2:]
    for c0 in range(0, rope_cols, d):
        a1 = y[:, c0:c0 + d // 2].copy()
        a2 = y[:, c0 + d // 2:c0 + d].copy()
        y[:, c0:c0 + d // 2] = a1 * cos - a2 * sin
        y[:, c0 + d // 2:c0 + d] = a2 * cos + a1 * sin
    return y


def causal_attention(qkv, hq, hkv, seq_len, causal=True, d=128):
    t = qkv.shape[0]
    q = qkv[:, :hq * d].reshape(t, hq, d)
    k = qkv[:, hq * d:(hq + hkv) * d].reshape(t, hkv, d)
    v = qkv[:, (hq + hkv) * d:].reshape(t, hkv, d)
    out = np.zeros((t, hq, d), np.float32)
    scale = np.float32(d ** -0.5)
    for s0 in range(0, t, seq_len):
        sl = slice(s0, s0 + seq_len)
        mask = np.triu(np.ones((seq_len, seq_len), bool), 1) if causal else None
        for h in range(hq):
            g = h // (hq // hkv)
            s = (q[sl, h] @ k[sl, g].T) * scale
            if causal:
                s = np.where(mask, -np.inf, s)
            s = s - s.max(axis=1, keepdims=True)
            p = np.exp(s)
            p /= p.sum(axis=1, keepdims=True)
            out[sl, h] = p @ v[sl, g]
    return bf(out.reshape(t, hq * d))


def llama_layer(x, g1, g2, rope, wqkv, wo, wg, wu, w2, hq, hkv, seq_len, eps=1e-5):
    """Per-rank weight shards (lists of length TP); returns (out, intermediates of rank 0).
    All tensors float32 arrays holding bf16 values."""
    tp = len(wqkv)
    xn = rmsnorm(x, g1, eps)
    parts, inter = [], {}
    for r in range(tp):
        qkv = bf(apply_rope(xn @ wqkv[r].T, rope, (hq + hkv) * 128, seq_len))
        att = causal_attention(qkv, hq, hkv, seq_len)
        parts.append(bf(att @ wo[r].T))
        if r == 0:
            inter.update(xn=xn, qkv=qkv, attn=att, o_part=parts[0])
    acc = parts[0].copy()
    for pr in parts[1:]:
        acc = acc + pr
    h = bf(acc + x)
    hn = rmsnorm(h, g2, eps)
    dparts = []
    for r in range(tp):
        gate, up = hn @ wg[r].T, hn @ wu[r].T
        act = bf(gate / (1.0 + np.exp(-gate)) * up)
        dparts.append(bf(act @ w2[r].T))
        if r == 0:
            inter.update(act=act, down_part=dparts[0])
    acc = dparts[0].copy()
    for pr in dparts[1:]:
        acc = acc + pr
    out = bf(acc + h)
    inter.update(h=h, hn=hn, out=out)
    return out, inter
