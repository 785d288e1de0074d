"""Oracle for the sequence-parallel attention scores (test infrastructure only).

BASELINE config 3 / SURVEY A13 is not in the reference; structurally it is the
reference's AllGather+GEMM (ovs/kernels/ag_gemm.py:20-94, oracle
ovs/kernels/oracles.py:12-15) with the gathered operand on the key side:
    scores_r[h] = Q_r[:, h, :] @ concat_s(K_s[:, h // (Hq/Hkv), :]).T
"""

from __future__ import annotations

import numpy as np

from .collectives import ref_allgather_gemm


def ref_ag_kv_scores(q_shards, k_shards, n_kv_heads: int):
    """Per rank: [Hq, S_local, S_total] (float64 for int inputs, else input dtype)."""
    outs = []
    for q in q_shards:
        q = np.asarray(q)
        hq = q.shape[1]
        group = hq // n_kv_heads
        per_head = []
        for h in range(hq):
            g = h // group
            k_g = [np.asarray(k)[:, g, :] for k in k_shards]
            # ref_allgather_gemm(A_shards, [B]) = concat(A) @ B.T  ->  transpose
            per_head.append(ref_allgather_gemm(k_g, [q[:, h, :]])[0].T)
        outs.append(np.stack(per_head))
    return outs


def ref_ag_kv_attention(q_shards, k_shards, v_shards, n_kv_heads: int, scale: float):
    """Per rank: O_r [S_local, Hq, d] = softmax(Q_r K_all^T * scale) V_all per head
    (non-causal), float64.  The K/V AllGather is the reference's ag_gemm gather."""
    k_all = np.concatenate([np.asarray(k, dtype=np.float64) for k in k_shards], axis=0)
    v_all = np.concatenate([np.asarray(v, dtype=np.float64) for v in v_shards], axis=0)
    outs = []
    for q in q_shards:
        q = np.asarray(q, dtype=np.float64)
        sl, hq, d = q.shape
        group = hq // n_kv_heads
        o = np.empty_like(q)
        for h in range(hq):
            g = h // group
            s = q[:, h, :] @ k_all[:, g, :].T * scale
            s = s - s.max(axis=1, keepdims=True)
            p = np.exp(s)
            o[:, h, :] = (p / p.sum(axis=1, keepdims=True)) @ v_all[:, g, :]
        outs.append(o)
    return outs
