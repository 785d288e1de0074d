"""Expert-parallel MoE: routing, dispatch and combine on the symmetric heap.

North-star row (d): routing counts and offsets computed on the device
(deterministic, bit-exact with oracle/moe.py), token rows packed with 16-byte
vector copies and scattered straight into the owners' receive buffers, and the
mirrored combine.  Layout conventions follow the reference:
  counts  [world, E]                     ovs/kernels/ag_moe.py:28-33
  receive expert-major / source rank / source order
                                         ovs/kernels/oracles.py:38-50
and the reference's own MoE operator is kept as a drop-in:
  ag_moe_group_gemm(token_shards, expert_weights, routing, ctx)
                                         ovs/kernels/ag_moe.py:20
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .context import WorkloadContext, WorkloadRun
from .shmem import SymmetricHeap, Team, tensor_from_ptr


def moe_route(logits: torch.Tensor, k: int, stream=None):
    """Top-k routing: (idx int32 [T,k], weights fp32 [T,k]); ties -> lower expert."""
    if logits.dtype != torch.float32 or not logits.is_cuda or logits.dim() != 2:
        raise ValueError("logits must be a 2-D float32 CUDA tensor")
    logits = logits.contiguous()
    t, e = logits.shape
    idx = torch.empty((t, k), dtype=torch.int32, device=logits.device)
    w = torch.empty((t, k), dtype=torch.float32, device=logits.device)
    s = stream or torch.cuda.current_stream(logits.device)
    _lib.call("tf_moe_topk", logits.data_ptr(), t, e, k, idx.data_ptr(), w.data_ptr(), s.cuda_stream)
    return idx, w


def moe_count(topk_idx: torch.Tensor, n_experts: int, stream=None):
    """This rank's routing row counts[E] and stable send positions [T,k]."""
    if topk_idx.dtype != torch.int32 or not topk_idx.is_cuda:
        raise ValueError("topk_idx must be an int32 CUDA tensor")
    topk_idx = topk_idx.contiguous()
    t, k = topk_idx.shape
    dev = topk_idx.device
    counts = torch.empty(n_experts, dtype=torch.int32, device=dev)
    pos = torch.empty((t, k), dtype=torch.int32, device=dev)
    nbytes = _lib.lib().tf_moe_count_scratch_bytes(t * k, n_experts)
    scratch = torch.empty(int(nbytes), dtype=torch.uint8, device=dev)
    s = stream or torch.cuda.current_stream(dev)
    _lib.call("tf_moe_count", topk_idx.data_ptr(), t, k, n_experts, counts.data_ptr(),
              pos.data_ptr(), scratch.data_ptr(), s.cuda_stream)
    return counts, pos


class ExpertParallelMoE:
    """Dispatch/combine for `n_experts` experts sharded over a team (rank d owns
    experts [d*E/w, (d+1)*E/w)).  Works for IPC teams (one rank per process) and
    for local teams (all ranks in this process; lists indexed by rank)."""

    def __init__(self, team: Team, n_experts: int, hidden: int, k: int, max_tokens: int,
                 max_recv: int | None = None):
        if n_experts % team.world:
            raise ValueError("n_experts must divide across ranks")
        if hidden % 8:
            raise ValueError("hidden must be a multiple of 8")
        self.team, self.E, self.H, self.k = team, n_experts, hidden, k
        self.max_tokens = max_tokens
        self.max_recv = max_recv if max_recv is not None else max_tokens * k * team.world
        self.state = {}
        for r in team.local_ranks():
            dev = team.devices[r]
            a = _lib.MoeArgs()
            a.hidden, a.k, a.n_experts, a.max_recv = hidden, k, n_experts, self.max_recv
            recv, yout = C.c_void_p(), C.c_void_p()
            with torch.cuda.device(dev):
                _lib.call("tf_moe_buffers", team.handle, r, C.byref(a), C.byref(recv), C.byref(yout))
            nbytes = self.max_recv * hidden * 2
            st = {
                "args": a,
                "recv": tensor_from_ptr(recv.value, nbytes, dev).view(torch.bfloat16).view(self.max_recv, hidden),
                "yout": tensor_from_ptr(yout.value, nbytes, dev).view(torch.bfloat16).view(self.max_recv, hidden),
                "counts": torch.zeros((team.world, n_experts), dtype=torch.int32, device=f"cuda:{dev}"),
                "recv_rows": torch.zeros(1, dtype=torch.int64, device=f"cuda:{dev}"),
                "pos": torch.empty((max_tokens, k), dtype=torch.int32, device=f"cuda:{dev}"),
                "dest": torch.empty((max_tokens, k), dtype=torch.int32, device=f"cuda:{dev}"),
            }
            self.state[r] = st

    # -------------------------------------------------------------- helpers
    def _fill(self, r, x, idx, w=None, out=None):
        st = self.state[r]
        a = st["args"]
        t = idx.shape[0]
        if t > self.max_tokens:
            raise ValueError(f"{t} tokens exceed max_tokens={self.max_tokens}")
        if idx.dtype != torch.int32 or idx.shape[1] != self.k:
            raise ValueError("topk_idx must be int32 [T, k]")
        a.tokens = t
        a.x = x.data_ptr() if x is not None else None
        a.topk_idx = idx.data_ptr()
        a.topk_w = w.data_ptr() if w is not None else None
        a.out = out.data_ptr() if out is not None else None
        a.counts = st["counts"].data_ptr()
        a.sorted_pos = st["pos"].data_ptr()
        a.dest_row = st["dest"].data_ptr()
        a.recv_rows = st["recv_rows"].data_ptr()
        return a

    def _ranks_args(self, x, idx):
        t = self.team
        if t.rank is not None or (t.world == 1 and isinstance(idx, torch.Tensor)):
            return {(t.rank or 0): (x, idx)}
        return {r: (x[r], idx[r]) for r in range(t.world)}

    def _drive(self, fn, per_rank):
        t = self.team
        for phase in (_lib.PHASE_PRE, _lib.PHASE_MAIN, _lib.PHASE_POST):
            for r, a in per_rank.items():
                with torch.cuda.device(t.devices[r]):
                    s = torch.cuda.current_stream(t.devices[r])
                    _lib.call(fn, t.handle, r, C.byref(a), phase, s.cuda_stream)

    # -------------------------------------------------------------- API
    def dispatch(self, x, topk_idx):
        """Scatter token rows to the experts' owners.  Returns, per local rank,
        the receive view [max_recv, H] (valid rows: recv_rows(r)).  After this
        call counts(r) holds the full [world, E] routing matrix."""
        items = self._ranks_args(x, topk_idx)
        for xx, ii in items.values():
            if xx.dtype != torch.bfloat16 or xx.shape[1] != self.H or not xx.is_contiguous():
                raise ValueError("x must be a contiguous bf16 [T, hidden] tensor")
        # the ctypes args hold raw pointers: keep the exact tensors they point into alive
        items = {r: (xx, ii.contiguous()) for r, (xx, ii) in items.items()}
        per = {r: self._fill(r, xx, ii) for r, (xx, ii) in items.items()}
        self._keep = items
        self._drive("tf_moe_dispatch", per)
        if isinstance(topk_idx, torch.Tensor):
            return self.state[next(iter(per))]["recv"]
        return [self.state[r]["recv"] for r in per]

    def _r(self, r):
        if r is not None:
            return r
        return self.team.rank if self.team.rank is not None else 0

    def counts(self, r=None):
        return self.state[self._r(r)]["counts"]

    def recv_rows(self, r=None) -> int:
        return int(self.state[self._r(r)]["recv_rows"].item())

    def dest_rows(self, r=None, tokens=None):
        st = self.state[self._r(r)]
        return st["dest"][: (tokens if tokens is not None else st["args"].tokens)]

    def expert_out(self, r=None):
        """[max_recv, H] bf16 buffer the experts write their outputs into (receive layout)."""
        return self.state[self._r(r)]["yout"]

    def combine(self, topk_idx, topk_w, out=None):
        """out[t] = sum_j w[t,j] * y_owner[row(t,j)] (fp32, slot order), bf16."""
        t = self.team
        single = t.rank is not None or (t.world == 1 and isinstance(topk_idx, torch.Tensor))
        if single:
            r = t.rank or 0
            items = {r: (topk_idx, topk_w, out)}
        else:
            items = {r: (topk_idx[r], topk_w[r], out[r] if out is not None else None)
                     for r in range(t.world)}
        per, outs = {}, {}
        for r, (ii, ww, oo) in items.items():
            if oo is None:
                oo = torch.empty((ii.shape[0], self.H), dtype=torch.bfloat16,
                                 device=f"cuda:{t.devices[r]}")
            outs[r] = oo
            items[r] = (ii.contiguous(), ww.contiguous().float(), oo)
            per[r] = self._fill(r, None, *items[r])
        self._keep2 = (items, outs)
        self._drive("tf_moe_combine", per)
        return outs[next(iter(outs))] if single else [outs[r] for r in range(t.world)]


# ---------------------------------------------------------------------- drop-in
def ag_moe_group_gemm(token_shards, expert_weights, routing, ctx: WorkloadContext) -> WorkloadRun:
    """Per rank r: expert-sorted gathered tokens times rank r's weight shards
    (ovs/kernels/ag_moe.py:20).  token_shards[r]: [rows_r, K] grouped by expert;
    expert_weights[r][e]: [N_per_rank, K]; routing [world, E] counts.

    Device path: copy-engine AllGather of the dynamic-size chunks into every
    rank's symmetric workspace (rank-major, ag_moe.py:99-115), one expert-major
    row permutation, then one tcgen05 GEMM per expert."""
    from . import kernels as K

    topo = ctx.topology
    world = topo.world_size
    routing = np.asarray(routing, dtype=np.int64)
    if routing.ndim != 2 or routing.shape[0] != world:
        raise ValueError(f"routing must be [world={world}, n_experts], got {routing.shape}")
    if np.any(routing < 0):
        raise ValueError("routing counts must be >= 0")
    n_experts = routing.shape[1]
    if len(token_shards) != world or len(expert_weights) != world:
        raise ValueError(f"need {world} token shards and weight sets")
    if len(expert_weights[0]) != n_experts:
        raise ValueError(f"need {n_experts} weight shards per rank")
    flat_w = [w for ws_ in expert_weights for w in ws_]
    K.check_dtype(*token_shards, *flat_w)
    k = token_shards[0].shape[1]
    n_per_rank = expert_weights[0][0].shape[0]
    for r in range(world):
        if tuple(token_shards[r].shape) != (int(routing[r].sum()), k):
            raise ValueError(f"rank {r} token shard {tuple(token_shards[r].shape)} inconsistent "
                             f"with routing sum {int(routing[r].sum())}")
        for w in expert_weights[r]:
            if tuple(w.shape) != (n_per_rank, k):
                raise ValueError("ragged expert weights")
    kp = (k + 7) // 8 * 8
    devices = K._devices_for(ctx, token_shards)
    pt = K._prepare(token_shards, devices, kp, 0)
    pw = [K._prepare(list(expert_weights[r]), [devices[r]] * n_experts, kp, 1) for r in range(world)]
    kp = pt.kdim
    if pt.kind == "exact":
        for p in pw:
            K._exact_bound_check(pt, p, k)
    odt = K._out_dtype(ctx.out_dtype, pt)

    rows_by_rank = routing.sum(axis=1)
    chunk_base = np.concatenate([[0], np.cumsum(rows_by_rank)])
    total = int(chunk_base[-1])
    tokens_per_expert = routing.sum(axis=0)
    expert_base = np.concatenate([[0], np.cumsum(tokens_per_expert)])
    in_rank_base = np.concatenate([np.zeros((world, 1), np.int64), np.cumsum(routing, axis=1)], axis=1)
    # expert-major row e,s,i <- rank-major row chunk_base[s] + in_rank_base[s,e] + i
    perm = np.empty(total, dtype=np.int64)
    pos = 0
    for e in range(n_experts):
        for s in range(world):
            c = int(routing[s, e])
            start = int(chunk_base[s] + in_rank_base[s, e])
            perm[pos:pos + c] = np.arange(start, start + c)
            pos += c

    row_bytes = kp * 2
    team = Team(world, devices, max(total, 1) * row_bytes + (1 << 20), 4 * world + 64)
    heap = SymmetricHeap(topo, team=team)
    ws = heap.alloc(max(total, 1) * row_bytes, align=1024)
    outs = []
    # AllGather: every rank's chunk into every rank's workspace at its rank-major offset
    for r in range(world):
        with torch.cuda.device(devices[r]):
            s = torch.cuda.current_stream(devices[r])
            for d in range(world):
                if rows_by_rank[r]:
                    heap.putmem(heap.symm_at(ws, d), int(chunk_base[r]) * row_bytes,
                                pt.tensors[r], from_pe=r, stream=s)
    for d in sorted(set(devices)):
        torch.cuda.synchronize(d)
    for r in range(world):
        dev = devices[r]
        with torch.cuda.device(dev):
            gathered = heap.view(ws, r, torch.bfloat16, (max(total, 1), kp))[:total]
            perm_t = torch.from_numpy(perm).to(f"cuda:{dev}")
            a_sorted = gathered.index_select(0, perm_t) if total else gathered
            out = torch.zeros((total, n_per_rank), dtype=odt, device=f"cuda:{dev}")
            for e in range(n_experts):
                lo, hi = int(expert_base[e]), int(expert_base[e + 1])
                if hi > lo and n_per_rank > 0:
                    K.gemm(a_sorted[lo:hi], pw[r].tensors[e], out[lo:hi], out_dtype=odt,
                           block_m=128, block_n=ctx.hw_block_n, group_m=ctx.group_m)
            outs.append(out)
    for d in sorted(set(devices)):
        torch.cuda.synchronize(d)
    team.check()
    return WorkloadRun([K._finish(o, pt) for o in outs], None, heap, {"workspace": ws})
