"""Sequence-parallel attention scores: AllGather-KV fused with Q.K^T.

BASELINE config 3 (32k context, SP=8, 64 query / 8 KV heads, d=128); SURVEY
§8(a) row A13.  Not in the reference -- structurally its ag_gemm
(ovs/kernels/ag_gemm.py:20-94) with the gathered operand on the N (key) side,
so it reuses the same symmetric-workspace pull protocol and the tcgen05 GEMM
with per-tile acquire waits on the *key* chunks and the gather swizzle applied
to key tiles.  GQA: query head h reads key head h // (Hq / Hkv).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from . import kernels as K
from .context import WorkloadContext, WorkloadRun
from .shmem import SymmetricHeap, Team


def _attn_args(q, k, scores, s_local, hq, hkv, d, out_dtype, block_m, block_n, group_m,
               num_gemm_sms, key_map):
    a = _lib.AttnArgs()
    a.q, a.k, a.scores = q.data_ptr(), k.data_ptr(), scores.data_ptr()
    a.s_local, a.hq, a.hkv, a.d = int(s_local), int(hq), int(hkv), int(d)
    a.out_dtype = _lib.TF_DTYPE_F32 if out_dtype == torch.float32 else _lib.TF_DTYPE_BF16
    a.block_m, a.block_n, a.group_m = int(block_m), int(block_n), int(group_m)
    a.num_gemm_sms = int(num_gemm_sms)
    a.swizzle = 1 if key_map is not None else 0
    a.key_tile_map = key_map.data_ptr() if key_map is not None else None
    return a


def ag_kv_scores(q_shards, k_shards, ctx: WorkloadContext, n_kv_heads: int | None = None) -> WorkloadRun:
    """Per rank r: scores_r = [Hq, S_local, S_total], scores_r[h] = Q_r[:, h] @ K_all[:, g(h)].T.

    q_shards[r]: [S_local, Hq, d]; k_shards[r]: [S_local, Hkv, d] (numpy int64 /
    float32 or torch bf16 CUDA, like the other drop-in operators)."""
    topo = ctx.topology
    world = topo.world_size
    if len(q_shards) != world or len(k_shards) != world:
        raise ValueError(f"need {world} shards per operand")
    K.check_dtype(*q_shards, *k_shards)
    sl, hq, d = q_shards[0].shape
    hkv = k_shards[0].shape[1] if n_kv_heads is None else n_kv_heads
    for q, k in zip(q_shards, k_shards):
        if tuple(q.shape) != (sl, hq, d) or tuple(k.shape) != (sl, hkv, d):
            raise ValueError("ragged q/k shards")
    if hq % hkv:
        raise ValueError("query heads must be a multiple of kv heads")
    devices = K._devices_for(ctx, q_shards)
    dp = (d + 7) // 8 * 8

    def flat(x, heads):  # per-head zero padding of the head dim to a multiple of 8
        if K._is_torch(x):
            x = torch.nn.functional.pad(x, (0, dp - d)) if dp != d else x
            return x.reshape(sl, heads * dp)
        x = np.asarray(x)
        if dp != d:
            x = np.concatenate([x, np.zeros((sl, heads, dp - d), x.dtype)], axis=2)
        return x.reshape(sl, heads * dp)

    pq = K._prepare([flat(q, hq) for q in q_shards], devices, hq * dp, split=False)
    pk = K._prepare([flat(k, hkv) for k in k_shards], devices, hkv * dp, split=False)
    K._exact_bound_check(pq, pk, d)
    odt = K._out_dtype(ctx.out_dtype, pq)
    st = sl * world
    team = Team(world, devices, 2 * st * hkv * dp * 2 + (1 << 20), 4 * world + 64)
    heap = SymmetricHeap(topo, team=team)
    outs, args, keep = [], {}, []
    for r in range(world):
        dev = devices[r]
        out = torch.empty((hq, sl, st), dtype=odt, device=f"cuda:{dev}")
        kmap = (K.tile_map_tensor(st, r, world, topo.nnodes, "ag_gemm", f"cuda:{dev}", ctx.hw_block_n)
                if ctx.swizzle and st > 0 else None)
        args[r] = _attn_args(pq.tensors[r], pk.tensors[r], out, sl, hq, hkv, dp, odt,
                             ctx.hw_block_m if ctx.hw_block_m != 512 else 256, ctx.hw_block_n,
                             ctx.group_m, ctx.num_gemm_sms, kmap)
        outs.append(out)
        keep.append(kmap)
    if sl > 0:
        for phase in (_lib.PHASE_PRE, _lib.PHASE_MAIN, _lib.PHASE_POST):
            for r in range(world):
                with torch.cuda.device(devices[r]):
                    s, cs = K._streams(team, r)
                    _lib.call("tf_ag_kv_scores", team.handle, r, C.byref(args[r]), phase,
                              K._ptr(s), K._ptr(cs))
    for dd in sorted(set(devices)):
        torch.cuda.synchronize(dd)
    team.check()
    return WorkloadRun([K._finish(o, pq) for o in outs], None, heap, {})


class AllGatherKVScores:
    """Reusable AG-KV.Q^T operator for a fixed shape (IPC team: one rank per process)."""

    def __init__(self, team: Team, s_local: int, hq: int, hkv: int, d: int, *,
                 out_dtype=torch.bfloat16, block_m: int = 256, block_n: int = 256,
                 group_m: int = 8, swizzle: bool = True):
        if d % 8 or hq % hkv:
            raise ValueError("d must be a multiple of 8 and hq a multiple of hkv")
        self.team, self.sl, self.hq, self.hkv, self.d = team, s_local, hq, hkv, d
        self.out_dtype, self.block_m, self.block_n, self.group_m = out_dtype, block_m, block_n, group_m
        st = s_local * team.world
        self.maps = {r: (K.tile_map_tensor(st, r, team.world, 1, "ag_gemm",
                                           f"cuda:{team.devices[r]}", block_n) if swizzle else None)
                     for r in team.local_ranks()}

    def forward(self, q, k, out=None):
        t = self.team
        r = t.rank or 0
        st = self.sl * t.world
        if out is None:
            out = torch.empty((self.hq, self.sl, st), dtype=self.out_dtype, device=q.device)
        a = _attn_args(q, k, out, self.sl, self.hq, self.hkv, self.d, out.dtype, self.block_m,
                       self.block_n, self.group_m, 0, self.maps[r])
        s, cs = torch.cuda.current_stream(), K.side_stream(q.device.index)
        _lib.call("tf_ag_kv_scores", t.handle, r, C.byref(a), _lib.PHASE_ALL, s.cuda_stream,
                  cs.cuda_stream)
        return out

    __call__ = forward


# ----------------------------------------------------------------- fused flash attention
def _fwd_args(q, k, v, out, s_local, hq, hkv, d, scale):
    a = _lib.AttnFwdArgs()
    a.q, a.k, a.v, a.out = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr()
    a.s_local, a.hq, a.hkv, a.d = int(s_local), int(hq), int(hkv), int(d)
    a.scale = float(scale)
    return a


def ag_kv_attention(q_shards, k_shards, v_shards, ctx: WorkloadContext, scale: float | None = None,
                    n_kv_heads: int | None = None) -> WorkloadRun:
    """Per rank r: O_r[:, h] = softmax(Q_r[:, h] . K_all[:, g(h)]^T * scale) . V_all[:, g(h)].

    Shards are torch bf16 CUDA tensors: q [S_local, Hq, 128], k/v [S_local, Hkv, 128]
    (S_local % 128 == 0).  The K/V AllGather is fused: each CTA waits per key chunk."""
    topo = ctx.topology
    world = topo.world_size
    if not (len(q_shards) == len(k_shards) == len(v_shards) == world):
        raise ValueError(f"need {world} shards per operand")
    K.check_dtype(*q_shards, *k_shards, *v_shards)
    if not K._is_torch(q_shards[0]):
        raise ValueError("ag_kv_attention takes torch bfloat16 CUDA tensors")
    sl, hq, d = q_shards[0].shape
    hkv = k_shards[0].shape[1] if n_kv_heads is None else n_kv_heads
    for q, k, v in zip(q_shards, k_shards, v_shards):
        if tuple(q.shape) != (sl, hq, d) or tuple(k.shape) != (sl, hkv, d) or tuple(v.shape) != (sl, hkv, d):
            raise ValueError("ragged q/k/v shards")
    if hq % hkv:
        raise ValueError("query heads must be a multiple of kv heads")
    if d != 128 or sl % 128:
        raise ValueError("the fused kernel needs head dim 128 and S_local % 128 == 0")
    scale = float(scale if scale is not None else d ** -0.5)
    devices = [t.device.index for t in q_shards]
    st = sl * world
    team = Team(world, devices, 2 * 2 * st * hkv * d * 2 + (1 << 20), 4 * world + 64)
    heap = SymmetricHeap(topo, team=team)
    outs = [torch.empty_like(q) for q in q_shards]
    # materialise the contiguous operands first and keep them alive for the launch:
    # the ctypes args hold raw pointers into exactly these tensors
    keep = [(q_shards[r].contiguous(), k_shards[r].contiguous(), v_shards[r].contiguous()) for r in range(world)]
    args = {r: _fwd_args(*keep[r], outs[r], sl, hq, hkv, d, scale) for r in range(world)}
    for phase in (_lib.PHASE_PRE, _lib.PHASE_MAIN, _lib.PHASE_POST):
        for r in range(world):
            with torch.cuda.device(devices[r]):
                s, cs = K._streams(team, r)
                _lib.call("tf_ag_kv_attention", team.handle, r, C.byref(args[r]), phase, K._ptr(s), K._ptr(cs))
    for dd in sorted(set(devices)):
        torch.cuda.synchronize(dd)
    team.check()
    del keep
    return WorkloadRun(outs, None, heap, {})


class AllGatherKVAttention:
    """Reusable fused AG-KV flash-attention forward (one rank per process, or a
    single-rank local team)."""

    def __init__(self, team: Team, s_local: int, hq: int, hkv: int, d: int = 128,
                 scale: float | None = None):
        if d != 128 or s_local % 128 or hq % hkv:
            raise ValueError("need d == 128, S_local % 128 == 0 and hq % hkv == 0")
        self.team, self.sl, self.hq, self.hkv, self.d = team, s_local, hq, hkv, d
        self.scale = float(scale if scale is not None else d ** -0.5)

    def forward(self, q, k, v, out=None):
        t = self.team
        if t.rank is None and t.world != 1:
            raise ValueError("use ag_kv_attention() for multi-rank local teams")
        r = t.rank or 0
        out = torch.empty_like(q) if out is None else out
        a = _fwd_args(q, k, v, out, self.sl, self.hq, self.hkv, self.d, self.scale)
        s, cs = torch.cuda.current_stream(), K.side_stream(q.device.index)
        _lib.call("tf_ag_kv_attention", t.handle, r, C.byref(a), _lib.PHASE_ALL, s.cuda_stream,
                  cs.cuda_stream)
        return out

    __call__ = forward
