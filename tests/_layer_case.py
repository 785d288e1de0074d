"""Shared inputs for the fused-layer tests (config 5 at parity-test sizes)."""

import numpy as np

from oracle import layer as OL
from paper_2605_02953_b200 import build_topology
from paper_2605_02953_b200 import layer as L


def make_case(tp, tokens=256, hidden=512, heads_q=8, heads_kv=2, ffn=1024, seq=None, seed=0):
    rng = np.random.default_rng(seed)
    seq = seq or tokens
    hq, hkv, f = heads_q // tp, heads_kv // tp, ffn // tp
    bf = OL.bf
    rn = lambda *s: rng.standard_normal(s).astype(np.float32)
    v = {
        "x": bf(rn(tokens, hidden)),
        "g_attn": bf(1.0 + 0.1 * rn(1, hidden)),
        "g_mlp": bf(1.0 + 0.1 * rn(1, hidden)),
        "rope": L.rope_table(seq),
        "w_qkv": [bf(rn((hq + 2 * hkv) * 128, hidden) * hidden ** -0.5) for _ in range(tp)],
        "w_o": [bf(rn(hidden, hq * 128) * (heads_q * 128) ** -0.5) for _ in range(tp)],
        "wg": [bf(rn(f, hidden) * hidden ** -0.5) for _ in range(tp)],
        "wu": [bf(rn(f, hidden) * hidden ** -0.5) for _ in range(tp)],
        "w_down": [bf(rn(hidden, f) * ffn ** -0.5) for _ in range(tp)],
    }
    prog = L.llama_layer_program(build_topology(tp, 1), tokens, hidden, heads_q, heads_kv, ffn, seq_len=seq)
    inputs = {k: v[k] for k in ("x", "g_attn", "g_mlp", "rope", "w_qkv", "w_o", "w_down")}
    inputs["w_gate_up"] = [L.interleave_gate_up(v["wg"][r], v["wu"][r]) for r in range(tp)]
    want, inter = OL.llama_layer(v["x"], v["g_attn"], v["g_mlp"], v["rope"], v["w_qkv"], v["w_o"],
                                 v["wg"], v["wu"], v["w_down"], hq, hkv, seq)
    return prog, inputs, want, inter
