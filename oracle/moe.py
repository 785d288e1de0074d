"""Oracle for expert-parallel routing, dispatch and combine (test infrastructure only).

The reference has no all-to-all; its MoE path is AllGather +
grouped GEMM (ovs/kernels/ag_moe.py:20-158).  What it does pin is the layout
convention, which the EP path here keeps:

* the routing count matrix is `[world, n_experts]`, entry (s, e) = number of
  rows source rank s sends to expert e (ag_moe.py:28-33, cli.py:193-202);
* a rank's token chunk is grouped by expert, ascending, and inside an expert
  keeps the source token order (ag_moe.py:_pull_engine + oracles.py:38-50);
* the receive side is expert-major, then source rank ascending, then the
  source's order (gather_tokens_by_expert, oracles.py:38-50).

For EP with `world` ranks, rank d owns experts [d*E/world, (d+1)*E/world) and
its receive buffer is exactly gather_tokens_by_expert restricted to those
experts.  Top-k selection is not in the reference ("parity unpinned"): the rule
fixed here is descending score, ties to the lower expert id, weights = softmax
over the selected scores in float32.  Combine sums the k weighted expert
outputs of a token in slot order j = 0..k-1 in float32.
"""

from __future__ import annotations

import numpy as np


def topk_route(logits: np.ndarray, k: int):
    """Deterministic top-k: (idx int32 [T,k], weights float32 [T,k])."""
    logits = np.asarray(logits, dtype=np.float32)
    t, e = logits.shape
    if not 1 <= k <= e:
        raise ValueError("need 1 <= k <= n_experts")
    # stable sort on (-score, expert id): lexsort keys are last-major
    order = np.lexsort((np.broadcast_to(np.arange(e), (t, e)), -logits), axis=1)[:, :k]
    sel = np.take_along_axis(logits, order, axis=1)
    z = np.exp(sel - sel[:, :1])
    w = (z / z.sum(axis=1, keepdims=True)).astype(np.float32)
    return order.astype(np.int32), w


def routing_counts(topk_idx_shards, n_experts: int) -> np.ndarray:
    """[world, E] int64 count matrix from per-rank top-k indices."""
    out = np.zeros((len(topk_idx_shards), n_experts), dtype=np.int64)
    for s, idx in enumerate(topk_idx_shards):
        out[s] = np.bincount(np.asarray(idx).reshape(-1), minlength=n_experts)[:n_experts]
    return out


def send_order(topk_idx: np.ndarray, n_experts: int):
    """A source rank's (token, slot) pairs grouped by expert then token order.

    Returns an int64 [T*k, 2] array of (token, slot).  This is the order in
    which a rank's rows appear in its expert-sorted chunk.
    """
    idx = np.asarray(topk_idx)
    t, k = idx.shape
    flat_e = idx.reshape(-1).astype(np.int64)
    tok = np.repeat(np.arange(t), k)
    slot = np.tile(np.arange(k), t)
    order = np.lexsort((slot, tok, flat_e))
    return np.stack([tok[order], slot[order]], axis=1)


def dispatch_layout(topk_idx_shards, n_experts: int, world: int):
    """Per destination rank: list of (src, token, slot) in receive-row order,
    plus per source rank: [T,k] receive row index on the owning rank."""
    if n_experts % world:
        raise ValueError("n_experts must divide across ranks")
    epr = n_experts // world
    counts = routing_counts(topk_idx_shards, n_experts)
    recv = [[] for _ in range(world)]
    slot_row = [np.full(np.asarray(i).shape, -1, dtype=np.int64) for i in topk_idx_shards]
    per_src_sorted = [send_order(i, n_experts) for i in topk_idx_shards]
    # position inside each source's expert-sorted chunk where expert e starts
    starts = np.zeros((world, n_experts + 1), dtype=np.int64)
    starts[:, 1:] = np.cumsum(counts, axis=1)
    for d in range(world):
        for e in range(d * epr, (d + 1) * epr):
            for s in range(world):
                for tok, sl in per_src_sorted[s][starts[s, e]:starts[s, e + 1]]:
                    slot_row[s][tok, sl] = len(recv[d])
                    recv[d].append((s, int(tok), int(sl)))
    return counts, recv, slot_row


def dispatch(x_shards, topk_idx_shards, n_experts: int):
    """Receive buffers per rank (expert-major / src-rank / token order)."""
    world = len(x_shards)
    _, recv, _ = dispatch_layout(topk_idx_shards, n_experts, world)
    out = []
    for d in range(world):
        rows = [np.asarray(x_shards[s])[t] for s, t, _ in recv[d]]
        h = np.asarray(x_shards[0]).shape[1]
        out.append(np.stack(rows) if rows else np.zeros((0, h), np.asarray(x_shards[0]).dtype))
    return out


def combine(expert_out_shards, topk_idx_shards, topk_w_shards, n_experts: int):
    """out_s[t] = sum_j w[t,j] * y_owner[row(t,j)], fp32, slot order j=0..k-1."""
    world = len(topk_idx_shards)
    _, _, slot_row = dispatch_layout(topk_idx_shards, n_experts, world)
    epr = n_experts // world
    outs = []
    for s in range(world):
        idx = np.asarray(topk_idx_shards[s])
        w = np.asarray(topk_w_shards[s], dtype=np.float32)
        t, k = idx.shape
        h = np.asarray(expert_out_shards[0]).shape[1]
        acc = np.zeros((t, h), dtype=np.float32)
        for j in range(k):
            for tok in range(t):
                owner = int(idx[tok, j]) // epr
                y = np.asarray(expert_out_shards[owner][slot_row[s][tok, j]], dtype=np.float32)
                acc[tok] += w[tok, j] * y
        outs.append(acc)
    return outs


def dispatch_layout_fast(topk_idx_shards, n_experts: int, world: int):
    """Vectorised dispatch_layout (same results, numpy lexsort instead of Python
    loops) for the full-size config-4 parity test: returns
    (counts [world, E], recv_src [world] of int64 arrays, recv_tok [world],
    slot_row [world] of [T, k] int64).  Receive order = expert, then source rank,
    then the source's (token, slot) order -- gather_tokens_by_expert
    (ovs/kernels/oracles.py:38-50) restricted to each owner's experts."""
    if n_experts % world:
        raise ValueError("n_experts must divide across ranks")
    epr = n_experts // world
    counts = routing_counts(topk_idx_shards, n_experts)
    es, ss, ts, ls = [], [], [], []
    for s, idx in enumerate(topk_idx_shards):
        idx = np.asarray(idx)
        t, k = idx.shape
        es.append(idx.reshape(-1).astype(np.int64))
        ss.append(np.full(t * k, s, np.int64))
        ts.append(np.repeat(np.arange(t, dtype=np.int64), k))
        ls.append(np.tile(np.arange(k, dtype=np.int64), t))
    e, s, tok, sl = (np.concatenate(v) if v else np.zeros(0, np.int64) for v in (es, ss, ts, ls))
    order = np.lexsort((sl, tok, s, e))
    e, s, tok, sl = e[order], s[order], tok[order], sl[order]
    owner = e // epr
    bounds = np.searchsorted(owner, np.arange(world + 1), side="left")
    pos = np.arange(e.size, dtype=np.int64) - bounds[owner]
    slot_row = [np.full(np.asarray(i).shape, -1, dtype=np.int64) for i in topk_idx_shards]
    for src in range(len(topk_idx_shards)):
        m = s == src
        slot_row[src][tok[m], sl[m]] = pos[m]
    recv_src = [s[bounds[d]:bounds[d + 1]] for d in range(world)]
    recv_tok = [tok[bounds[d]:bounds[d + 1]] for d in range(world)]
    return counts, recv_src, recv_tok, slot_row
