"""Sequential oracles for the fused collectives (test infrastructure only).

Restates /root/reference/pkg/src/overlapsim/kernels/oracles.py:
  ref_allgather_gemm       oracles.py:12-15
  ref_reduce_scatter       oracles.py:18-27   (rank-ordered sum, then slice)
  ref_allreduce            oracles.py:30-35
  gather_tokens_by_expert  oracles.py:38-50   (expert-major, then source rank)
  ref_group_gemm           oracles.py:53-69
plus `compare`, the max-norm relative error of ovs/cli.py:253-271.

Inputs are numpy arrays (int64 for exact mode, float32/float64 otherwise).  The
GPU path computes in bf16 with fp32 accumulation; callers upcast the exact bf16
inputs to float32/float64 before calling these.
"""

from __future__ import annotations

import numpy as np


def ref_allgather_gemm(a_shards, b_shards):
    full = np.concatenate([np.asarray(a) for a in a_shards], axis=0)
    return [full @ np.asarray(b).T for b in b_shards]


def ref_reduce_scatter(input_shards, weight_shards):
    world = len(input_shards)
    acc = None
    for x, w in zip(input_shards, weight_shards):
        part = np.asarray(x) @ np.asarray(w).T
        acc = part if acc is None else acc + part
    rows = acc.shape[0]
    if rows % world:
        raise ValueError(f"M={rows} not divisible by world {world}")
    per = rows // world
    return [acc[r * per:(r + 1) * per].copy() for r in range(world)]


def ref_allreduce(a_shards, b_shards):
    acc = None
    for a, b in zip(a_shards, b_shards):
        part = np.asarray(a) @ np.asarray(b).T
        acc = part if acc is None else acc + part
    return acc


def gather_tokens_by_expert(token_shards, routing):
    routing = np.asarray(routing, dtype=np.int64)
    world, n_exp = routing.shape
    starts = np.zeros((world, n_exp + 1), dtype=np.int64)
    starts[:, 1:] = np.cumsum(routing, axis=1)
    blocks = [np.asarray(token_shards[s])[starts[s, e]:starts[s, e + 1]]
              for e in range(n_exp) for s in range(world)]
    return np.concatenate(blocks, axis=0)


def ref_group_gemm(token_shards, expert_weights, routing):
    routing = np.asarray(routing, dtype=np.int64)
    gathered = gather_tokens_by_expert(token_shards, routing)
    edges = np.zeros(routing.shape[1] + 1, dtype=np.int64)
    edges[1:] = np.cumsum(routing.sum(axis=0))
    outs = []
    for per_rank in expert_weights:
        cols = np.asarray(per_rank[0]).shape[0]
        y = np.zeros((gathered.shape[0], cols), dtype=gathered.dtype)
        for e, w in enumerate(per_rank):
            lo, hi = edges[e], edges[e + 1]
            if hi > lo:
                y[lo:hi] = gathered[lo:hi] @ np.asarray(w).T
        outs.append(y)
    return outs


def compare(got, want) -> float:
    """Max-norm relative error, the reference CLI's verification metric."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    diff = float(np.max(np.abs(got - want), initial=0.0))
    scale = float(np.max(np.abs(want), initial=0.0)) or 1.0
    return diff / scale
