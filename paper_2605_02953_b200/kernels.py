"""Fused collective operators behind the reference's operator API.

Drop-in entry points (same names, argument order and errors as the reference):
  ag_gemm(a_shards, b_shards, ctx)                          ovs/kernels/ag_gemm.py:20
  gemm_rs(input_shards, weight_shards, ctx,
          assume_full_mesh_links=True)                      ovs/kernels/gemm_rs.py:31
All ranks' shards are passed in one call (ag_gemm.py:24-25).  Shards may be
torch bf16 CUDA tensors (production: bf16 output unless ctx.out_dtype) or the
reference's numpy float32 / int64 arrays (parity: computed in bf16 with fp32
accumulation and fp32 output, returned as numpy of the input dtype; int64
"exact mode" inputs must be bf16-exact integers so results are bit-identical).

Per-rank persistent operators for one-process-per-GPU use (torchrun) and for
benchmarking: `AllGatherGemm`, `GemmReduceScatter`, and the single-GPU core
`gemm()`.  Everything runs through libtilefuse; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _lib
from .context import SUPPORTED_NUMPY, WorkloadContext, WorkloadRun
from .shmem import SigHandle, SymmetricHeap, Team

BM = 128
_side_streams: dict[int, torch.cuda.Stream] = {}


def side_stream(device: int) -> torch.cuda.Stream:
    s = _side_streams.get(device)
    if s is None:
        with torch.cuda.device(device):
            s = torch.cuda.Stream(device=device)
        _side_streams[device] = s
    return s


# ----------------------------------------------------------------- input prep
class _Prepared:
    def __init__(self, tensors, kind, np_dtype, k_orig, kdim):
        self.tensors = tensors
        self.kind = kind          # "torch" | "exact" | "float"
        self.np_dtype = np_dtype
        self.k = k_orig
        self.kdim = kdim          # K of the device operands (6*kp for split float32)


def _is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


def check_dtype(*arrays):
    """Reference check_dtype (context.py:67-74) extended with torch bf16."""
    first = arrays[0]
    if _is_torch(first):
        for a in arrays:
            if not _is_torch(a) or a.dtype != torch.bfloat16:
                raise ValueError(f"unsupported dtype {getattr(a, 'dtype', type(a))}; "
                                 "torch inputs must be bfloat16")
            if not a.is_cuda:
                raise ValueError("torch inputs must be CUDA tensors (there is no CPU path)")
        return torch.bfloat16
    dt = np.asarray(first).dtype
    if dt not in SUPPORTED_NUMPY:
        raise ValueError(f"unsupported dtype {dt}; use float32 or int64 (exact mode), or torch bfloat16")
    for a in arrays[1:]:
        if _is_torch(a) or np.asarray(a).dtype != dt:
            raise ValueError(f"mixed dtypes: {dt} vs {getattr(a, 'dtype', type(a))}")
    return dt


def _pad_k(t: torch.Tensor, kp: int) -> torch.Tensor:
    if t.shape[1] == kp and t.stride(1) == 1 and (t.stride(0) * 2) % 16 == 0 and t.data_ptr() % 16 == 0:
        return t
    out = torch.zeros((t.shape[0], kp), dtype=t.dtype, device=t.device)
    out[:, : t.shape[1]] = t
    return out


def split_f32(x: torch.Tensor, kp: int, role: int) -> torch.Tensor:
    """fp32 [rows, k] CUDA tensor -> the 6-term bf16 operand [rows, 6*kp] (role 0 = A,
    1 = B) whose bf16 GEMM reproduces the fp32 product (tf_prep.cu)."""
    x = x.contiguous()
    rows, k = x.shape
    out = torch.empty((rows, 6 * kp), dtype=torch.bfloat16, device=x.device)
    with torch.cuda.device(x.device):
        _lib.call("tf_split_f32_bf16x3", x.data_ptr(), rows, k, k, out.data_ptr(), kp, role,
                  torch.cuda.current_stream(x.device).cuda_stream)
    return out


def _prepare(shards, devices, kp: int, role: int = 0, split: bool = True) -> _Prepared:
    """Device operands for one side of a GEMM.  float32 numpy inputs (the
    reference's float contract) become the 6-term split operand (split=False:
    rounded to bf16, for operators whose kernels index K per head); int64 "exact"
    inputs must be bf16-exact integers and stay one term."""
    dt = check_dtype(*shards)
    k = shards[0].shape[1]
    if dt is torch.bfloat16:
        return _Prepared([_pad_k(s, kp) for s in shards], "torch", None, k, kp)
    kind = "exact" if dt == np.int64 else "float"
    out = []
    for s, dev in zip(shards, devices):
        arr = np.asarray(s)
        if kind == "exact" or not split:
            if kind == "exact" and arr.size and np.abs(arr).max() > 256:
                raise ValueError("exact mode needs integers with |x| <= 256 (exact in bf16)")
            t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).to(torch.bfloat16)
            t = _pad_k(t, kp) if kp != k else t
            out.append(t.to(f"cuda:{dev}"))
        else:
            f = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).to(f"cuda:{dev}")
            out.append(split_f32(f, kp, role))
    return _Prepared(out, kind, dt, k, 6 * kp if (kind == "float" and split) else kp)


def _exact_bound_check(prep_a: _Prepared, prep_b: _Prepared, k: int, extra_terms: int = 1):
    if prep_a.kind != "exact":
        return
    amax = max((float(t.float().abs().max()) for t in prep_a.tensors if t.numel()), default=0.0)
    bmax = max((float(t.float().abs().max()) for t in prep_b.tensors if t.numel()), default=0.0)
    if amax * bmax * k * extra_terms >= 2 ** 24:
        raise ValueError("exact mode: |sum| may exceed 2^24, fp32 accumulation would not be exact")


def _finish(out: torch.Tensor, prep: _Prepared):
    if prep.kind == "torch":
        return out
    host = out.float().cpu().numpy()
    if prep.kind == "exact":
        return np.rint(host).astype(np.int64)
    return host.astype(np.float32)


def _out_dtype(ctx_out: str | None, prep: _Prepared) -> torch.dtype:
    if prep.kind != "torch":
        return torch.float32
    return torch.float32 if ctx_out == "f32" else torch.bfloat16


def _tf_dtype(t: torch.dtype) -> int:
    return _lib.TF_DTYPE_F32 if t == torch.float32 else _lib.TF_DTYPE_BF16


def tile_map_tensor(m: int, rank: int, world: int, nnodes: int, mode: str, device,
                    block_m: int = BM) -> torch.Tensor:
    """Gather (mode 'ag_gemm') / scatter ('gemm_rs') map from the C library, on device."""
    tiles = (m + block_m - 1) // block_m
    buf = (C.c_int32 * max(tiles, 1))()
    _lib.call("tf_tile_map", int(m), int(rank), int(world), int(nnodes), int(block_m),
              0 if mode == "ag_gemm" else 1, buf, tiles)
    host = np.frombuffer(bytes(buf), dtype=np.int32)[:tiles].copy()
    return torch.from_numpy(host).to(device)


def _tile_map_or_none(m: int, rank: int, world: int, nnodes: int, mode: str, device, block_m: int):
    """The swizzle only orders tiles (results do not depend on it): when the hardware
    tile is too coarse for the node ranges of a multi-node topology (e.g. 16 rows on
    2 nodes with 128-row tiles) the identity order is used."""
    from .errors import ProtocolError
    try:
        return tile_map_tensor(m, rank, world, nnodes, mode, device, block_m)
    except ProtocolError:
        return None


def tile_map_host(m: int, rank: int, world: int, nnodes: int, block_m: int, mode: str) -> np.ndarray:
    tiles = (m + block_m - 1) // block_m
    buf = (C.c_int32 * max(tiles, 1))()
    _lib.call("tf_tile_map", int(m), int(rank), int(world), int(nnodes), int(block_m),
              0 if mode == "ag_gemm" else 1, buf, tiles)
    return np.frombuffer(bytes(buf), dtype=np.int32)[:tiles].astype(np.int64)


def _args(a, b, c, m, n, k, *, out_dtype, block_n, group_m, num_gemm_sms, num_comm_sms,
          swizzle, tile_map, fuse_scatter=0, reduce_order="ring", ldc=None,
          block_m=BM) -> _lib.GemmArgs:
    g = _lib.GemmArgs()
    g.a = a.data_ptr() if a is not None else None
    g.b = b.data_ptr() if b is not None else None
    g.c = c.data_ptr() if c is not None else None
    g.m, g.n, g.k = int(m), int(n), int(k)
    g.lda = int(a.stride(0)) if a is not None else int(k)
    g.ldb = int(b.stride(0)) if b is not None else int(k)
    g.ldc = int(ldc if ldc is not None else (c.stride(0) if c is not None else n))
    g.out_dtype = _tf_dtype(out_dtype)
    g.block_m, g.block_n, g.block_k = int(block_m), int(block_n), 64
    g.group_m = int(group_m)
    g.num_gemm_sms = int(num_gemm_sms)
    g.num_comm_sms = int(num_comm_sms)
    g.swizzle = 1 if (swizzle and tile_map is not None) else 0
    g.fuse_scatter = 1 if fuse_scatter else 0
    g.reduce_order = _lib.TF_REDUCE_RING if reduce_order == "ring" else _lib.TF_REDUCE_ASCENDING
    g.tile_map = tile_map.data_ptr() if tile_map is not None else None
    return g


def _streams(team: Team, rank: int):
    dev = team.devices[rank]
    s = torch.cuda.current_stream(dev)
    if team.distinct_devices:
        return s, side_stream(dev)
    return s, None


def _ptr(s) -> int | None:
    return None if s is None else s.cuda_stream


def _drive(team: Team, fn_name: str, per_rank_args: dict, ranks, extra=()):
    """Run PRE for all local ranks, then MAIN, then POST, then FINAL
    (single-process teams: PEs sharing a stream never wait on later work)."""
    for phase in (_lib.PHASE_PRE, _lib.PHASE_MAIN, _lib.PHASE_POST, _lib.PHASE_FINAL):
        for r in ranks:
            dev = team.devices[r]
            with torch.cuda.device(dev):
                s, cs = _streams(team, r)
                _lib.call(fn_name, team.handle, r, C.byref(per_rank_args[r]), *extra,
                          phase, _ptr(s), _ptr(cs))


# ----------------------------------------------------------------- core GEMM
def gemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None, *,
         out_dtype: torch.dtype = torch.bfloat16, block_m: int = 512, block_n: int = 256,
         group_m: int = 8, num_sms: int = 0, tile_map: torch.Tensor | None = None,
         stream=None) -> torch.Tensor:
    """C = A @ B.T on one GPU with the tcgen05 kernel (bf16 in, fp32 accumulate).
    block_m=256 uses a CTA pair per tile (cta_group::2), 128 one CTA; a tile_map
    must be expressed in tiles of block_m rows."""
    check_dtype(a, b)
    if a.dim() != 2 or b.dim() != 2 or a.shape[1] != b.shape[1]:
        raise ValueError(f"need A [M,K], B [N,K]; got {tuple(a.shape)} and {tuple(b.shape)}")
    m, k = a.shape
    n = b.shape[0]
    if a.stride(1) != 1 or b.stride(1) != 1:
        raise ValueError("A and B must be K-contiguous")
    if out is None:
        out = torch.empty((m, n), dtype=out_dtype, device=a.device)
    g = _args(a, b, out, m, n, k, out_dtype=out.dtype, block_n=block_n, group_m=group_m,
              num_gemm_sms=num_sms, num_comm_sms=0, swizzle=tile_map is not None,
              tile_map=tile_map, block_m=block_m)
    s = stream if stream is not None else torch.cuda.current_stream(a.device)
    _lib.call("tf_gemm", C.byref(g), s.cuda_stream)
    return out


# ----------------------------------------------------------------- AllGather + GEMM
# Teams (symmetric heaps + flags) of the drop-in entry points are cached per (op,
# world, devices, heap size, slots), so repeated calls of the same shape reuse the
# peer mappings and workspaces instead of rebuilding them (the reference builds a
# heap per call, ag_gemm.py:35; here that is a one-time cost).  Epoch-valued flags make
# back-to-back reuse safe.  TF_TEAM_CACHE=0 restores a fresh team per call.
_TEAM_CACHE: "dict" = {}
_TEAM_CACHE_MAX = 4


def _cached_team(op, world, devices, heap_bytes, slots):
    if os.environ.get("TF_TEAM_CACHE", "1") == "0":
        return Team(world, devices, heap_bytes, slots)
    key = (op, world, tuple(devices), int(heap_bytes), int(slots))
    team = _TEAM_CACHE.pop(key, None)
    if team is None:
        team = Team(world, devices, heap_bytes, slots)
        while len(_TEAM_CACHE) >= _TEAM_CACHE_MAX:  # evict the least recently used
            _TEAM_CACHE.pop(next(iter(_TEAM_CACHE))).close()
    _TEAM_CACHE[key] = team  # most recently used last
    return team


def ag_gemm(a_shards, b_shards, ctx: WorkloadContext) -> WorkloadRun:
    """Per rank r: C_r = concat(a_0..a_{w-1}) @ b_r.T, shape [M, N_per_rank]."""
    topo = ctx.topology
    world = topo.world_size
    if len(a_shards) != world or len(b_shards) != world:
        raise ValueError(f"need {world} shards per operand")
    check_dtype(*a_shards, *b_shards)
    m_per_rank, k = a_shards[0].shape
    n_per_rank = b_shards[0].shape[0]
    for a, b in zip(a_shards, b_shards):
        if tuple(a.shape) != (m_per_rank, k):
            raise ValueError(f"ragged A shards: {tuple(a.shape)} vs {(m_per_rank, k)}")
        if tuple(b.shape) != (n_per_rank, k):
            raise ValueError(f"B shard must be [N_per_rank, K]-shaped, got {tuple(b.shape)}")
    m = m_per_rank * world
    kp = (k + 7) // 8 * 8
    devices = _devices_for(ctx, a_shards)
    pa = _prepare(a_shards, devices, kp, 0)
    pb = _prepare(b_shards, devices, kp, 1)
    _exact_bound_check(pa, pb, k)
    odt = _out_dtype(ctx.out_dtype, pa)
    kp = pa.kdim
    if ctx.ag_pull == "sm" and m_per_rank > 0 and n_per_rank > 0:
        # in-kernel gather: num_comm_sms pull-engine CTAs + the GEMM in one launch per rank
        from .moe import _agmoe_heap_bytes
        bm = 256 if ctx.hw_block_m >= 256 else 128
        n_pad = max((n_per_rank + 7) // 8 * 8, 8)
        team = _cached_team("ag_gemm_pull", world, devices, _agmoe_heap_bytes(m, kp, 1, world, bm), 4 * world + 64)
        heap = SymmetricHeap(topo, team=team)
        op = AllGatherGemm(team, m, kp, n_pad, out_dtype=odt, block_m=bm, block_n=ctx.hw_block_n,
                           num_gemm_sms=ctx.num_gemm_sms, swizzle=ctx.swizzle,
                           num_comm_sms=max(1, ctx.num_comm_sms))
        wts = []
        for r in range(world):
            w = pb.tensors[r]
            if n_pad != n_per_rank:
                w = torch.cat([w, torch.zeros((n_pad - n_per_rank, kp), dtype=w.dtype, device=w.device)])
            wts.append(w.contiguous())
        outs = [torch.zeros((m, n_pad), dtype=odt, device=f"cuda:{devices[r]}") for r in range(world)]
        op.forward([pa.tensors[r] for r in range(world)], wts, out=outs)
        for d in sorted(set(devices)):
            torch.cuda.synchronize(d)
        team.check()
        return WorkloadRun([_finish(o[:, :n_per_rank], pa) for o in outs], None, heap, {})
    heap_bytes = 2 * m * kp * 2 + (1 << 20)
    team = _cached_team("ag_gemm", world, devices, heap_bytes, 4 * world + 64)
    heap = SymmetricHeap(topo, team=team)
    outs, args, keep = [], {}, []
    for r in range(world):
        dev = devices[r]
        out = torch.empty((m, n_per_rank), dtype=odt, device=f"cuda:{dev}")
        tm = (_tile_map_or_none(m, r, world, topo.nnodes, "ag_gemm", f"cuda:{dev}", ctx.hw_block_m)
              if ctx.swizzle else None)
        a = pa.tensors[r]
        args[r] = _args(a, pb.tensors[r], out, m, n_per_rank, kp, out_dtype=odt,
                        block_n=ctx.hw_block_n, group_m=ctx.group_m,
                        num_gemm_sms=ctx.num_gemm_sms, num_comm_sms=ctx.num_comm_sms,
                        swizzle=ctx.swizzle, tile_map=tm, block_m=ctx.hw_block_m)
        outs.append(out)
        keep.append(tm)
    if m_per_rank > 0 and n_per_rank > 0:
        _drive(team, "tf_ag_gemm", args, range(world))
    for d in sorted(set(devices)):
        torch.cuda.synchronize(d)
    team.check()
    del keep
    return WorkloadRun([_finish(o, pa) for o in outs], None, heap, {})


# ----------------------------------------------------------------- GEMM + ReduceScatter
def gemm_rs(input_shards, weight_shards, ctx: WorkloadContext,
            assume_full_mesh_links: bool = True) -> WorkloadRun:
    """Per rank r: rows r of sum_w(input_w @ weight_w.T), shape [M_per_rank, N].

    The unfused reduction follows the reference's summation tree
    (gemm_rs.py:199-319): per node a fold in reduce_visit_order -- or, with
    `assume_full_mesh_links=False`, the neighbour-ring order of _scatter_ring --
    then a fold of the node partials.  On NVSwitch every peer is one hop, so the
    data still moves as one pull per peer; only the arithmetic order changes."""
    topo = ctx.topology
    world = topo.world_size
    if len(input_shards) != world or len(weight_shards) != world:
        raise ValueError(f"need {world} shards per operand")
    check_dtype(*input_shards, *weight_shards)
    m, k_local = input_shards[0].shape
    n = weight_shards[0].shape[0]
    if m % world != 0:
        raise ValueError(f"M={m} must divide evenly across {world} ranks")
    for inp, w in zip(input_shards, weight_shards):
        if tuple(inp.shape) != (m, k_local) or tuple(w.shape) != (n, k_local):
            raise ValueError("ragged shards")
    mpr = m // world
    kp = (k_local + 7) // 8 * 8
    devices = _devices_for(ctx, input_shards)
    px = _prepare(input_shards, devices, kp, 0)
    pw = _prepare(weight_shards, devices, kp, 1)
    _exact_bound_check(px, pw, k_local, extra_terms=world)
    odt = _out_dtype(ctx.out_dtype, px)
    kp = px.kdim
    esz = 4 if odt == torch.float32 else 2
    ld = (n + 7) // 8 * 8
    heap_bytes = m * ld * esz + (1 << 20)
    num_pid_m = (m + BM - 1) // BM
    team = _cached_team(f"gemm_rs:{bool(ctx.fuse_scatter)}", world, devices, heap_bytes, num_pid_m + 64)
    heap = SymmetricHeap(topo, team=team)
    outs, args, keep = [], {}, []
    for r in range(world):
        dev = devices[r]
        out = torch.empty((mpr, n), dtype=odt, device=f"cuda:{dev}")
        tm = (_tile_map_or_none(m, r, world, topo.nnodes, "gemm_rs", f"cuda:{dev}", ctx.hw_block_m)
              if ctx.swizzle else None)
        args[r] = _args(px.tensors[r], pw.tensors[r], out, m, n, kp, out_dtype=odt,
                        block_n=ctx.hw_block_n, group_m=ctx.group_m,
                        num_gemm_sms=ctx.num_gemm_sms, num_comm_sms=ctx.num_comm_sms,
                        swizzle=ctx.swizzle, tile_map=tm, fuse_scatter=ctx.fuse_scatter,
                        reduce_order=ctx.reduce_order, block_m=ctx.hw_block_m)
        args[r].nnodes = int(topo.nnodes)
        args[r].ring_links = 0 if assume_full_mesh_links else 1
        outs.append(out)
        keep.append(tm)
    if mpr > 0 and n > 0:
        _drive(team, "tf_gemm_rs", args, range(world))
    for d in sorted(set(devices)):
        torch.cuda.synchronize(d)
    team.check()
    # counters live right after the reserved slots; expose them for hygiene checks
    handles = {"counters": SigHandle(base=world + 1, nslots=num_pid_m)}
    return WorkloadRun([_finish(o, px) for o in outs], None, heap, handles)


def _devices_for(ctx: WorkloadContext, shards) -> list[int]:
    if ctx.devices is not None:
        return [int(d) for d in ctx.devices]
    if _is_torch(shards[0]):
        return [s.device.index for s in shards]
    world = ctx.topology.world_size
    ndev = torch.cuda.device_count()
    if ndev == 0:
        raise RuntimeError("no CUDA device: the tilefuse operators have no CPU path")
    return list(range(world)) if ndev >= world else [0] * world


# ----------------------------------------------------------------- persistent per-rank ops
class AllGatherGemm:
    """Reusable AllGather+GEMM for a fixed shape over a team.

    For an IPC team (torchrun) call `forward(a_local, b_local, out)`; for a local
    team pass lists indexed by rank.  The workspace and flags are created once
    in the team heap; each call is one epoch."""

    def __init__(self, team: Team, m: int, k: int, n_local: int, *, out_dtype=torch.bfloat16,
                 block_m: int = 512, block_n: int = 256, group_m: int = 8,
                 num_gemm_sms: int = 0, swizzle: bool = True, nnodes: int = 1,
                 num_comm_sms: int = 0):
        if k % 8:
            raise ValueError("K must be a multiple of 8")
        self.team, self.m, self.k, self.n = team, m, k, n_local
        # num_comm_sms > 0: the gather runs INSIDE the GEMM launch -- that many pull-engine
        # CTAs copy the peers' chunks ((rank+i)%w order) over NVLink into the workspace and
        # release per-source arrival counters the GEMM tiles wait on (the reference's
        # _pull_engine process, ag_gemm.py:55-69, as SM work).  This is the grouped
        # AG-GEMM kernel with a single group (tf_ag_moe_group_gemm, E = 1).
        self._pull = None
        if num_comm_sms > 0:
            from .moe import AgMoeGroupGemm
            if m % team.world:
                raise ValueError("M must divide across ranks")
            self._pull = AgMoeGroupGemm(team, 1, n_local, k, m, block_m=256 if block_m >= 256 else 128,
                                        block_n=block_n, num_gemm_sms=num_gemm_sms,
                                        num_comm_sms=num_comm_sms, swizzle=swizzle, out_dtype=out_dtype)
            self._routing = np.full((team.world, 1), m // team.world, dtype=np.int64)
        self.out_dtype = out_dtype
        self.block_m, self.block_n = block_m, block_n
        # a raster group must not span more than one gathered chunk: with the gather
        # swizzle the first group is then this rank's own rows, so the first wave of
        # tiles needs no remote data (TP8 at 512-row tiles: 2 row tiles per chunk)
        if team.world > 1 and swizzle:
            group_m = max(1, min(group_m, (m // team.world) // block_m))
        self.group_m, self.num_gemm_sms = group_m, num_gemm_sms
        self.maps = {r: (tile_map_tensor(m, r, team.world, nnodes, "ag_gemm",
                                         f"cuda:{team.devices[r]}", block_m) if swizzle else None)
                     for r in team.local_ranks()}

    def _args(self, r, a, b, out):
        return _args(a, b, out, self.m, self.n, self.k, out_dtype=out.dtype, block_n=self.block_n,
                     group_m=self.group_m, num_gemm_sms=self.num_gemm_sms, num_comm_sms=0,
                     swizzle=self.maps[r] is not None, tile_map=self.maps[r],
                     block_m=self.block_m)

    def forward(self, a, b, out=None):
        t = self.team
        if self._pull is not None:
            if isinstance(b, torch.Tensor):
                return self._pull(self._routing, a, b.unsqueeze(0), out=out)
            return self._pull(self._routing, list(a), [x.unsqueeze(0) for x in b], out=out)
        if t.rank is not None or (t.world == 1 and isinstance(a, torch.Tensor)):
            r = t.rank or 0
            if out is None:
                out = torch.empty((self.m, self.n), dtype=self.out_dtype, device=a.device)
            g = self._args(r, a, b, out)
            s, cs = torch.cuda.current_stream(), side_stream(a.device.index)
            _lib.call("tf_ag_gemm", t.handle, r, C.byref(g), _lib.PHASE_ALL, s.cuda_stream, cs.cuda_stream)
            return out
        outs = out or [torch.empty((self.m, self.n), dtype=self.out_dtype,
                                   device=f"cuda:{t.devices[r]}") for r in range(t.world)]
        args = {r: self._args(r, a[r], b[r], outs[r]) for r in range(t.world)}
        _drive(t, "tf_ag_gemm", args, range(t.world))
        return outs

    __call__ = forward


class GemmReduceScatter:
    """Reusable fused GEMM+ReduceScatter for a fixed shape over a team."""

    def __init__(self, team: Team, m: int, k_local: int, n: int, *, out_dtype=torch.bfloat16,
                 block_m: int = 512, block_n: int = 256, group_m: int = 8, num_gemm_sms: int = 0,
                 num_comm_sms: int = 8, swizzle: bool = True, fuse_scatter: bool = True,
                 reduce_order: str = "ascending", nnodes: int = 1):
        if k_local % 8:
            raise ValueError("K must be a multiple of 8")
        if m % team.world:
            raise ValueError("M must divide evenly across ranks")
        self.team, self.m, self.k, self.n = team, m, k_local, n
        self.out_dtype = out_dtype
        self.block_m, self.block_n, self.group_m = block_m, block_n, group_m
        self.num_gemm_sms, self.num_comm_sms = num_gemm_sms, num_comm_sms
        self.fuse, self.order = fuse_scatter, reduce_order
        self.maps = {r: (tile_map_tensor(m, r, team.world, nnodes, "gemm_rs",
                                         f"cuda:{team.devices[r]}", block_m) if swizzle else None)
                     for r in team.local_ranks()}

    def _args(self, r, x, w, out):
        return _args(x, w, out, self.m, self.n, self.k, out_dtype=out.dtype, block_n=self.block_n,
                     group_m=self.group_m, num_gemm_sms=self.num_gemm_sms,
                     num_comm_sms=self.num_comm_sms, swizzle=self.maps[r] is not None,
                     tile_map=self.maps[r], fuse_scatter=self.fuse, reduce_order=self.order,
                     block_m=self.block_m)

    def forward(self, x, w, out=None):
        t = self.team
        mpr = self.m // t.world
        if t.rank is not None or (t.world == 1 and isinstance(x, torch.Tensor)):
            r = t.rank or 0
            if out is None:
                out = torch.empty((mpr, self.n), dtype=self.out_dtype, device=x.device)
            g = self._args(r, x, w, out)
            s, cs = torch.cuda.current_stream(), side_stream(x.device.index)
            _lib.call("tf_gemm_rs", t.handle, r, C.byref(g), _lib.PHASE_ALL, s.cuda_stream, cs.cuda_stream)
            return out
        outs = out or [torch.empty((mpr, self.n), dtype=self.out_dtype,
                                   device=f"cuda:{t.devices[r]}") for r in range(t.world)]
        args = {r: self._args(r, x[r], w[r], outs[r]) for r in range(t.world)}
        _drive(t, "tf_gemm_rs", args, range(t.world))
        return outs

    __call__ = forward


# ----------------------------------------------------------------- GEMM + AllReduce
def gemm_allreduce(a_shards, b_shards, ctx: WorkloadContext, use_multimem_st: bool | None = None) -> WorkloadRun:
    """Per rank: sum_w(a_w @ b_w.T), shape [M, N], identical on every rank
    (ovs/kernels/gemm_ar.py:25).  use_multimem_st selects the two-shot protocol
    (owner reduce + P2P broadcast), else one-shot (every rank pull-reduces)."""
    topo = ctx.topology
    world = topo.world_size
    if topo.nnodes != 1:
        raise ValueError("allreduce workload requires a single node (node-team reduction)")
    if len(a_shards) != world or len(b_shards) != world:
        raise ValueError(f"need {world} shards per operand")
    check_dtype(*a_shards, *b_shards)
    m, k = a_shards[0].shape
    n = b_shards[0].shape[0]
    if n % ctx.block_n != 0:
        raise ValueError(f"N={n} must be divisible by block_n={ctx.block_n}")
    for a, b in zip(a_shards, b_shards):
        if tuple(a.shape) != (m, k) or tuple(b.shape) != (n, k):
            raise ValueError("ragged shards")
    two_shot = ctx.use_multimem_st if use_multimem_st is None else use_multimem_st
    kp = (k + 7) // 8 * 8
    devices = _devices_for(ctx, a_shards)
    pa = _prepare(a_shards, devices, kp, 0)
    pb = _prepare(b_shards, devices, kp, 1)
    _exact_bound_check(pa, pb, k, extra_terms=world)
    odt = _out_dtype(ctx.out_dtype, pa)
    kp = pa.kdim
    esz = 4 if odt == torch.float32 else 2
    ld = (n + 7) // 8 * 8
    nblocks = (m + 127) // 128
    team = Team(world, devices, 2 * m * ld * esz + (1 << 20), 2 * nblocks + 64)  # may bind an NVLS region
    if two_shot and team.distinct_devices and world > 1 and os.environ.get("TF_NVLS", "1") != "0":
        # two-shot through the switch (multimem.ld_reduce + multimem.st) when the
        # box exposes NVLS; otherwise the P2P owner-reduce + broadcast below
        team.enable_nvls(2 * m * ld * esz + (4 << 20))
    heap = SymmetricHeap(topo, team=team)
    outs, args = [], {}
    for r in range(world):
        out = torch.empty((m, n), dtype=odt, device=f"cuda:{devices[r]}")
        args[r] = _args(pa.tensors[r], pb.tensors[r], out, m, n, kp, out_dtype=odt,
                        block_n=ctx.hw_block_n, group_m=ctx.group_m, num_gemm_sms=ctx.num_gemm_sms,
                        num_comm_sms=ctx.num_comm_sms, swizzle=False, tile_map=None,
                        block_m=ctx.hw_block_m)
        outs.append(out)
    if m > 0 and n > 0:
        _drive(team, "tf_gemm_ar", args, range(world), extra=(1 if two_shot else 0,))
    for d in sorted(set(devices)):
        torch.cuda.synchronize(d)
    team.check()
    # teardown like the reference (gemm_ar.py:128-153): every flag reads 0 afterwards
    tile_ready = SigHandle(base=world + 1, nslots=nblocks)
    mst_sig = SigHandle(base=world + 1 + nblocks, nslots=nblocks)
    for r in range(world):
        with torch.cuda.device(devices[r]):
            heap.reset_signals(tile_ready, r)
            heap.reset_signals(mst_sig, r)
    for d in sorted(set(devices)):
        torch.cuda.synchronize(d)
    return WorkloadRun([_finish(o, pa) for o in outs], None, heap,
                       {"tile_ready": tile_ready, "mst_sig": mst_sig})


class GemmAllReduce:
    """Reusable fused GEMM+AllReduce for a fixed shape over a team (one rank per
    process, or a single-rank local team)."""

    def __init__(self, team: Team, m: int, k: int, n: int, *, out_dtype=torch.bfloat16,
                 block_m: int = 512, block_n: int = 256, group_m: int = 8, num_comm_sms: int = 8,
                 two_shot: bool = False):
        if k % 8:
            raise ValueError("K must be a multiple of 8")
        self.team, self.m, self.k, self.n = team, m, k, n
        self.out_dtype, self.block_m, self.block_n, self.group_m = out_dtype, block_m, block_n, group_m
        self.num_comm_sms, self.two_shot = num_comm_sms, two_shot

    def forward(self, a, b, out=None):
        t = self.team
        if t.rank is None and t.world != 1:
            raise ValueError("GemmAllReduce drives one rank per process; use gemm_allreduce() for local teams")
        r = t.rank or 0
        if out is None:
            out = torch.empty((self.m, self.n), dtype=self.out_dtype, device=a.device)
        g = _args(a, b, out, self.m, self.n, self.k, out_dtype=out.dtype, block_n=self.block_n,
                  group_m=self.group_m, num_gemm_sms=0, num_comm_sms=self.num_comm_sms,
                  swizzle=False, tile_map=None, block_m=self.block_m)
        s, cs = torch.cuda.current_stream(), side_stream(a.device.index)
        _lib.call("tf_gemm_ar", t.handle, r, C.byref(g), 1 if self.two_shot else 0, _lib.PHASE_ALL,
                  s.cuda_stream, cs.cuda_stream)
        return out

    __call__ = forward
