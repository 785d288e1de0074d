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
import math

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
                 max_recv: int | None = None, capacity_factor: float | None = None):
        """Receive capacity per rank: `max_recv` rows if given, else
        ceil(capacity_factor * max_tokens * k) rows (balanced routing delivers
        max_tokens * k rows to each rank on average), else the worst case
        max_tokens * k * world (every token of every source to one rank), which can
        never overflow.  A dispatch that would write past the capacity skips those
        rows and `team.check()` raises (TF_ERR_INVALID, "receive buffer overflow")."""
        if n_experts % team.world:
            raise ValueError("n_experts must divide across ranks")
        if hidden % 8:
            raise ValueError("hidden must be a multiple of 8")
        if max_recv is not None and capacity_factor is not None:
            raise ValueError("give max_recv or capacity_factor, not both")
        if capacity_factor is not None and not capacity_factor > 0:
            raise ValueError("capacity_factor must be > 0")
        self.team, self.E, self.H, self.k = team, n_experts, hidden, k
        self.max_tokens = max_tokens
        if max_recv is None:
            worst = max_tokens * k * team.world
            max_recv = worst if capacity_factor is None else min(worst, math.ceil(capacity_factor * max_tokens * k))
        self.max_recv = int(max_recv)
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
    def _fill(self, r, x, idx, w=None, out=None, logits=None):
        st = self.state[r]
        a = st["args"]
        t = idx.shape[0]
        if t > self.max_tokens:
            raise ValueError(f"{t} tokens exceed max_tokens={self.max_tokens}")
        if idx.dtype != torch.int32 or idx.shape[1] != self.k:
            raise ValueError("topk_idx must be int32 [T, k]")
        a.logits = logits.data_ptr() if logits is not None else None
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

    def _phases(self):
        """PRE and MAIN are one call (one launch for the dispatch) when every rank
        has its own GPU; ranks sharing a GPU need every PRE enqueued before any
        MAIN waits on it."""
        t = self.team
        if t.rank is not None or t.world == 1 or t.distinct_devices:
            return (_lib.PHASE_PRE | _lib.PHASE_MAIN, _lib.PHASE_POST)
        return (_lib.PHASE_PRE, _lib.PHASE_MAIN, _lib.PHASE_POST)

    def _drive(self, fn, per_rank):
        t = self.team
        for phase in self._phases():
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

    def route_dispatch(self, x, logits):
        """Top-k routing (as moe_route: ties -> lower expert) fused into the
        dispatch launch.  Returns (recv, topk_idx, topk_w), per local rank as
        lists for a local team with several ranks."""
        items = self._ranks_args(x, logits)
        per, keep, res = {}, {}, {}
        for r, (xx, lg) in items.items():
            if xx.dtype != torch.bfloat16 or xx.shape[1] != self.H or not xx.is_contiguous():
                raise ValueError("x must be a contiguous bf16 [T, hidden] tensor")
            if lg.dtype != torch.float32 or lg.dim() != 2 or lg.shape[0] != xx.shape[0] or lg.shape[1] != self.E:
                raise ValueError(f"logits must be float32 [T, {self.E}]")
            lg = lg.contiguous()
            idx = torch.empty((lg.shape[0], self.k), dtype=torch.int32, device=lg.device)
            w = torch.empty((lg.shape[0], self.k), dtype=torch.float32, device=lg.device)
            keep[r] = (xx, lg, idx, w)
            per[r] = self._fill(r, xx, idx, w, None, logits=lg)
            res[r] = (self.state[r]["recv"], idx, w)
        self._keep = keep
        self._drive("tf_moe_dispatch", per)
        if isinstance(logits, torch.Tensor):
            return res[next(iter(per))]
        return [res[r] for r in per]

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


# ---------------------------------------------------------------------- AG + grouped GEMM
def _agmoe_heap_bytes(max_rows: int, kdim: int, n_experts: int, world: int, block_m: int) -> int:
    """Symmetric bytes tf_ag_moe_group_gemm carves per PE (two call parities of the
    expert-major rows plus the tile/piece tables)."""
    al = lambda x: (x + 1023) // 1024 * 1024  # noqa: E731
    rows = al(max(max_rows, 1) * kdim * 2) if world > 1 else 0
    slots = -(-max_rows // block_m) + n_experts
    tab = al(slots * 16 + world * (n_experts + 1) * 4 + world * n_experts * 4)
    return 2 * (rows + tab) + (1 << 20)


class AgMoeGroupGemm:
    """Persistent AllGather + grouped GEMM (the reference's ag_moe_group_gemm,
    ovs/kernels/ag_moe.py:20-142) for one team: a local team (all ranks in this
    process, lists indexed by rank) or an IPC team (one rank per process).

    Each call: routing [world, E] host counts (the same on every rank), this
    rank's expert-grouped token rows [rows_r, K] bf16 and its stacked expert
    weights [E, N, K] bf16 -> [total_rows, N] expert-major output.  One launch per
    rank runs the pull engine (num_comm_sms CTAs) and the grouped tcgen05 GEMM,
    whose tiles wait only on the source ranks their rows come from."""

    def __init__(self, team: Team, n_experts: int, n: int, k: int, max_rows: int, *,
                 block_m: int = 128, block_n: int = 256, num_gemm_sms: int = 0,
                 num_comm_sms: int = 0, swizzle: bool = True, out_dtype=torch.bfloat16):
        if n % 8 or k % 8:
            raise ValueError("n and k must be multiples of 8")
        if block_m not in (128, 256) or block_n not in (128, 256):
            raise ValueError("block_m must be 128 or 256, block_n 128 or 256")
        self.team, self.E, self.n, self.k, self.max_rows = team, n_experts, n, k, max_rows
        self.block_m, self.block_n = block_m, block_n
        self.num_gemm_sms, self.num_comm_sms, self.swizzle = num_gemm_sms, num_comm_sms, swizzle
        self.out_dtype = out_dtype
        self._keep = None

    def _args(self, tokens, weights, out, routing_np) -> _lib.AgMoeArgs:
        a = _lib.AgMoeArgs()
        a.tokens = tokens.data_ptr() if tokens is not None and tokens.numel() else None
        a.weights = weights.data_ptr()
        a.out = out.data_ptr()
        a.routing = routing_np.ctypes.data
        a.n_experts, a.n, a.k, a.max_rows = self.E, self.n, self.k, self.max_rows
        a.lda = int(tokens.stride(0)) if tokens is not None and tokens.numel() else self.k
        a.ldo = int(out.stride(0))
        a.out_dtype = _lib.TF_DTYPE_F32 if out.dtype == torch.float32 else _lib.TF_DTYPE_BF16
        a.block_m, a.block_n = self.block_m, self.block_n
        a.num_gemm_sms, a.num_comm_sms = self.num_gemm_sms, self.num_comm_sms
        a.swizzle = 1 if self.swizzle else 0
        return a

    def __call__(self, routing, tokens, weights, out=None, phases=_lib.PHASE_ALL):
        """Local team: tokens/weights/out are lists indexed by rank; IPC team: this
        rank's tensors.  Returns the output(s)."""
        t = self.team
        routing_np = np.ascontiguousarray(np.asarray(routing, dtype=np.int64))
        if routing_np.shape != (t.world, self.E):
            raise ValueError(f"routing must be [{t.world}, {self.E}], got {routing_np.shape}")
        total = int(routing_np.sum())
        single = not isinstance(tokens, (list, tuple))
        ranks = list(t.local_ranks())
        toks = {ranks[0]: tokens} if single else dict(enumerate(tokens))
        wts = {ranks[0]: weights} if single else dict(enumerate(weights))
        outs = {}
        for r in ranks:
            w = wts[r]
            if w.dtype != torch.bfloat16 or tuple(w.shape) != (self.E, self.n, self.k) or not w.is_contiguous():
                raise ValueError(f"weights must be contiguous bf16 [{self.E}, {self.n}, {self.k}]")
            tk = toks[r]
            rows = int(routing_np[r].sum())
            if tk is not None and (tk.dtype != torch.bfloat16 or tuple(tk.shape) != (rows, self.k)):
                raise ValueError(f"rank {r} tokens must be bf16 [{rows}, {self.k}]")
            o = None if out is None else (out if single else out[r])
            if o is None:
                o = torch.empty((total, self.n), dtype=self.out_dtype, device=w.device)
            outs[r] = o
        args = {r: self._args(toks[r], wts[r], outs[r], routing_np) for r in ranks}
        self._keep = (routing_np, toks, wts, outs, args)
        for ph in (_lib.PHASE_PRE, _lib.PHASE_MAIN):
            if not ph & phases:
                continue
            for r in ranks:
                dev = t.devices[r]
                with torch.cuda.device(dev):
                    s = torch.cuda.current_stream(dev)
                    _lib.call("tf_ag_moe_group_gemm", t.handle, r, C.byref(args[r]), ph, s.cuda_stream)
        return outs[ranks[0]] if single else [outs[r] for r in range(t.world)]


# ---------------------------------------------------------------------- drop-in
def ag_moe_group_gemm(token_shards, expert_weights, routing, ctx: WorkloadContext) -> WorkloadRun:
    """Per rank r: expert-sorted gathered tokens times rank r's weight shards
    (ovs/kernels/ag_moe.py:20).  token_shards[r]: [rows_r, K] grouped by expert;
    expert_weights[r][e]: [N_per_rank, K]; routing [world, E] counts.

    Device path (tf_ag_moe_group_gemm): per rank ONE launch in which pull-engine
    CTAs gather the peers' dynamic-size chunks (source (rank+i)%w at step i,
    ag_moe.py:99-117) straight into expert-major rows of the symmetric
    workspace, while the grouped tcgen05 GEMM walks the swizzle_ag_moe schedule
    and acquire-waits, per tile, only the source ranks [segment_start,
    segment_end] its rows come from (ag_moe.py:120-142).  Output rows are
    expert-major."""
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
    kdim = pt.kdim
    if pt.kind == "exact":
        for p in pw:
            K._exact_bound_check(pt, p, k)
    odt = K._out_dtype(ctx.out_dtype, pt)
    total = int(routing.sum())
    n_pad = max((n_per_rank + 7) // 8 * 8, 8)
    block_m = 256 if ctx.hw_block_m >= 256 else 128
    stacked = []
    for r in range(world):
        wr = torch.zeros((n_experts, n_pad, kdim), dtype=torch.bfloat16, device=f"cuda:{devices[r]}")
        for e in range(n_experts):
            wr[e, :n_per_rank] = pw[r].tensors[e]
        stacked.append(wr)
    team = Team(world, devices, _agmoe_heap_bytes(total, kdim, n_experts, world, block_m), 4 * world + 64)
    heap = SymmetricHeap(topo, team=team)
    op = AgMoeGroupGemm(team, n_experts, n_pad, kdim, max(total, 1), block_m=block_m,
                        block_n=ctx.hw_block_n, num_gemm_sms=ctx.num_gemm_sms,
                        num_comm_sms=ctx.num_comm_sms, swizzle=ctx.swizzle, out_dtype=odt)
    toks = [pt.tensors[r] if pt.tensors[r].shape[0] else None for r in range(world)]
    outs = [torch.zeros((total, n_pad), dtype=odt, device=f"cuda:{devices[r]}") for r in range(world)]
    if total and n_per_rank:
        op(routing, toks, stacked, out=outs)
    for d in sorted(set(devices)):
        torch.cuda.synchronize(d)
    team.check()
    return WorkloadRun([K._finish(o[:, :n_per_rank], pt) for o in outs], None, heap, {})
