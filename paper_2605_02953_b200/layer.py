"""bf16 transformer-layer ops for the task-level megakernel (BASELINE config 5).

The reference's megakernel (ovs/megakernel/) ships three fp32 builders
(`linear`, `add`, `allreduce`, builders.py:168-236) and an open registry
(`register_task_builder`, builders.py:75-80) for more.  This module registers
the ops a Llama layer needs -- `rmsnorm`, `attention` (causal GQA flash
attention over a fused QKV buffer) and `allreduce_residual` -- and a bf16 mode
of `linear` (tcgen05 128x256 tiles with a plain, RoPE or SiLU*up epilogue),
all under the reference's planner contract (LayerPlan / TileSpec /
InputDependencyDesc / OutputTilingDesc, region-intersection dependencies).

`LayerRunner` executes a bf16 program on the device with one persistent launch
of `tf_layer_megakernel_run` (csrc/tf_layer.cu); `llama_layer_program` builds
the TP-sharded Llama-3 layer graph:

    xn  = rmsnorm(x, g_attn)                     tiles: 32-row blocks
    qkv = linear(xn, Wqkv) + RoPE(q, k)          128 x 256 tiles
    att = attention(qkv)  (causal, GQA)          (128-query tile, head)
    op  = linear(att, Wo)                        partial sums (K sharded over TP)
    h, hn = allreduce_residual(op, x)            h = sum_rank op + x, hn = rmsnorm(h) fused
    act = linear(hn, W13) -> silu(gate) * up     gate/up rows interleaved per 128
    dp  = linear(act, W2)                        partial sums
    out = allreduce_residual(dp, h)
"""

from __future__ import annotations

import ctypes as C
import os
import struct

import numpy as np

from . import megakernel as MK
from .errors import BuildError

try:  # numpy has no native bfloat16; ml_dtypes provides the storage type
    import ml_dtypes as _mld
    bfloat16 = np.dtype(_mld.bfloat16)
except ImportError:  # pragma: no cover - the image ships ml_dtypes
    bfloat16 = None

if bfloat16 is not None:
    MK.DTYPE_TAGS[bfloat16] = 2
    MK.TAG_DTYPES[2] = bfloat16

LAYER_OP_CODES = {"rmsnorm": 1, "linear": 2, "attention": 3, "allreduce_residual": 4}
EPILOGUES = {"none": 0, "rope": 1, "silu_mul": 2}
HEAD_DIM = 128
BLOCK_M, BLOCK_N = 256, 256
CFG_INTS = 16


def is_bf16(t) -> bool:
    return bfloat16 is not None and np.dtype(t.dtype) == bfloat16


def _f32_bits(v: float) -> int:
    return struct.unpack("<i", struct.pack("<f", float(v)))[0]


# ---------------------------------------------------------------------- planners
def plan_linear_bf16(io, config) -> MK.LayerPlan:
    """bf16 linear: y[m, n] = x[m, k] . w[n, k]^T on 256 x 256 tiles (two tcgen05
    M=128 x N=256 halves sharing each B stage).
    epilogue "rope": third input = rope table [seq, 128] fp32 (cos | sin), RoPE on
    output columns [0, rope_cols); "silu_mul": w rows interleaved per 128 (gate
    block, up block), y[m, n/2] = silu(gate) * up."""
    ins, (y,) = io[0], io[1]
    x, w = ins[0], ins[1]
    m, k = x.shape
    n, wk = w.shape
    cfg = {"block_m": BLOCK_M, "block_n": BLOCK_N, "block_k": 64, "epilogue": "none", **config}
    if (cfg["block_m"], cfg["block_n"]) != (BLOCK_M, BLOCK_N):
        raise BuildError("bf16 linear tiles are 256 x 256 (two tcgen05 M=128, N=256 halves)")
    epi = cfg["epilogue"]
    if epi not in EPILOGUES:
        raise BuildError(f"unknown linear epilogue {epi!r}")
    if wk != k or k % 64 or n % 8:
        raise BuildError(f"linear shapes: x{x.shape} w{w.shape} (k % 64 == 0, n % 8 == 0)")
    want_y = (m, n // 2) if epi == "silu_mul" else (m, n)
    if y.shape != want_y:
        raise BuildError(f"linear output {y.shape}, expected {want_y}")
    if epi == "silu_mul" and n % BLOCK_N:
        raise BuildError("silu_mul needs n % 256 == 0 (gate/up blocks of 128 rows)")
    if epi == "rope":
        if len(ins) != 3 or ins[2].shape[1] != HEAD_DIM:
            raise BuildError("rope epilogue needs a [seq, 128] fp32 rope table as third input")
        if cfg.get("rope_cols", n) % HEAD_DIM:
            raise BuildError("rope_cols must be a multiple of the head dim")
    elif len(ins) != 2:
        raise BuildError("linear takes (x, w)")
    tm_n, tn_n = -(-m // BLOCK_M), -(-n // BLOCK_N)
    tiles = []
    # emission order = grouped raster (swizzle_2d, ovs/swizzle.py:76-88) so the tiles one
    # wave of round-robin queues runs share group_m A panels and ~grid/group_m B panels in
    # L2; tile ids stay row-major (the dependency contract)
    gm = max(1, int(cfg.get("group_m", os.environ.get("TF_LAYER_GROUP_M", 8))))
    for step in range(tm_n * tn_n):
        grp, r = divmod(step, gm * tn_n)
        rows = min(tm_n - grp * gm, gm)
        tm, tn = grp * gm + r % rows, r // rows
        if True:
            deps = [MK.InputDependencyDesc(x, start_indices=(tm * BLOCK_M, 0),
                                           data_sizes=(min(BLOCK_M, m - tm * BLOCK_M), k)),
                    MK.InputDependencyDesc(w, start_indices=(tn * BLOCK_N, 0),
                                           data_sizes=(min(BLOCK_N, n - tn * BLOCK_N), k))]
            tiles.append(MK.TileSpec(tm * tn_n + tn, tuple(deps)))
    out_tile = (BLOCK_M, BLOCK_N // 2) if epi == "silu_mul" else (BLOCK_M, BLOCK_N)
    return MK.LayerPlan("linear", io, cfg, tm_n * tn_n, tiles, {y.name: MK.OutputTilingDesc(out_tile)})


def plan_rmsnorm(io, config) -> MK.LayerPlan:
    (x, g), (y,) = io[0], io[1]
    rows, cols = x.shape
    if y.shape != x.shape or g.shape != (1, cols) or cols % 8:
        raise BuildError(f"rmsnorm shapes: x{x.shape} g{g.shape} y{y.shape} (cols % 8 == 0)")
    cfg = {"block_rows": 32, "eps": 1e-5, **config}
    br = cfg["block_rows"]
    n = -(-rows // br)
    tiles = [MK.TileSpec(t, (MK.InputDependencyDesc(x, start_indices=(t * br, 0),
                                                    data_sizes=(min(br, rows - t * br), cols)),
                             MK.InputDependencyDesc(g, require_full=True)))
             for t in range(n)]
    return MK.LayerPlan("rmsnorm", io, cfg, n, tiles, {y.name: MK.OutputTilingDesc((br, cols))})


def plan_allreduce_residual(io, config) -> MK.LayerPlan:
    """y = (x_0 + ... + x_{w-1}) + res over the team (fp32, ascending rank), bf16.
    With `norm_gain=<[1, cols] tensor>` the following RMSNorm is fused in: a second
    output yn = y * rsqrt(mean(y^2) + eps) * gain (one pass over the rows).
    two_shot (default): row block b is reduced only by rank b % world, which stores
    the result into every rank's copy over P2P and releases the tile on every
    rank's scoreboard (reduce-scatter + all-gather traffic, 2 (w-1)/w of the data
    per rank, instead of every rank reading all w partials).
    Tiles are row blocks; each tile waits on the producer tiles of its rows on
    every rank (the reference's allreduce waits on the whole input, builders.py:222)."""
    (x, res), outs = io[0], io[1]
    y = outs[0]
    if not (x.shape == res.shape == y.shape) or x.shape[1] % 8:
        raise BuildError(f"allreduce_residual shapes must match (cols % 8 == 0): {x.shape} {res.shape} {y.shape}")
    cfg = {"block_rows": 32, "eps": 1e-5, "norm_gain": None, "two_shot": True, **config}
    if (cfg["norm_gain"] is None) != (len(outs) == 1):
        raise BuildError("allreduce_residual: a second output needs norm_gain (and vice versa)")
    if cfg["norm_gain"] is not None and (cfg["norm_gain"].shape != (1, x.shape[1]) or outs[1].shape != y.shape):
        raise BuildError("allreduce_residual norm: gain [1, cols] and yn shaped like y")
    rows, cols = x.shape
    br = cfg["block_rows"]
    n = -(-rows // br)
    tiles = []
    for t in range(n):
        reg = dict(start_indices=(t * br, 0), data_sizes=(min(br, rows - t * br), cols))
        tiles.append(MK.TileSpec(t, (MK.InputDependencyDesc(x, **reg), MK.InputDependencyDesc(res, **reg))))
    return MK.LayerPlan("allreduce_residual", io, cfg, n, tiles,
                        {o.name: MK.OutputTilingDesc((br, cols)) for o in outs})


def plan_attention(io, config) -> MK.LayerPlan:
    """Flash-attention forward over a fused qkv [T, (hq + 2 hkv) * 128] buffer
    (q heads, then k heads, then v heads), out [T, hq * 128]; sequences of
    `seq_len` rows, causal by default.  Tile (i, p) = query rows [128 i, 128 i + 128)
    of heads [p * np, p * np + np) (np = heads_per_task, 2 by default when the GQA
    group is even), tile id i * hq / np + p; emitted longest-first (descending i) so
    the static round-robin queues start with the long causal rows."""
    (qkv,), (o,) = io[0], io[1]
    cfg = {"heads_q": None, "heads_kv": None, "seq_len": None, "causal": True, **config}
    hq, hkv = cfg["heads_q"], cfg["heads_kv"]
    t_rows = qkv.shape[0]
    seq = cfg["seq_len"] or t_rows
    cfg["seq_len"] = seq
    cfg.setdefault("scale", HEAD_DIM ** -0.5)
    if not hq or not hkv or hq % hkv:
        raise BuildError("attention needs heads_q % heads_kv == 0")
    if qkv.shape[1] != (hq + 2 * hkv) * HEAD_DIM or o.shape != (t_rows, hq * HEAD_DIM):
        raise BuildError(f"attention shapes: qkv{qkv.shape} o{o.shape} for hq={hq} hkv={hkv} d=128")
    if seq % 128 or t_rows % seq:
        raise BuildError("seq_len must be a multiple of 128 dividing the token count")
    tps = seq // 128
    grp = hq // hkv
    # two heads of one KV group per task when possible: they share every K/V tile and
    # the device overlaps one head's softmax with the other head's MMAs
    npt = cfg.get("heads_per_task") or (2 if grp % 2 == 0 else 1)
    if npt not in (1, 2) or (npt == 2 and grp % 2):
        raise BuildError("heads_per_task must be 1, or 2 with an even GQA group")
    cfg["heads_per_task"] = npt
    per_row = hq // npt
    tiles = []
    # causal emission order: "shortest_first" (default: early query tiles need only the
    # first QKV rows, so attention starts while QKV is still running and the O
    # projection follows row by row; +0.7% at config 5 in a same-box A/B) or
    # "longest_first" (classic LPT balance of the static queues)
    order = cfg.get("order", os.environ.get("TF_ATTN_ORDER", "shortest_first"))
    if order not in ("longest_first", "shortest_first"):
        raise BuildError(f"unknown attention order {order!r}")
    cfg["order"] = order
    sign = -1 if order == "longest_first" else 1
    for i in sorted(range(t_rows // 128), key=lambda i: (sign * (i % tps), i)) if cfg["causal"] else range(t_rows // 128):
        kv0 = (i // tps) * tps
        n_kv = i - kv0 + 1 if cfg["causal"] else tps
        for hp in range(per_row):
            h = hp * npt
            g = h // grp
            deps = (
                MK.InputDependencyDesc(qkv, start_indices=(i * 128, h * HEAD_DIM), data_sizes=(128, npt * HEAD_DIM)),
                MK.InputDependencyDesc(qkv, start_indices=(kv0 * 128, (hq + g) * HEAD_DIM),
                                       data_sizes=(n_kv * 128, HEAD_DIM)),
                MK.InputDependencyDesc(qkv, start_indices=(kv0 * 128, (hq + hkv + g) * HEAD_DIM),
                                       data_sizes=(n_kv * 128, HEAD_DIM)),
            )
            tiles.append(MK.TileSpec(i * per_row + hp, deps))
    return MK.LayerPlan("attention", io, cfg, (t_rows // 128) * per_row, tiles,
                        {o.name: MK.OutputTilingDesc((128, npt * HEAD_DIM))})


_ref_plan_linear = MK.get_task_builder("linear").plan


def _plan_linear_any(io, config):
    """The reference's fp32 linear (builders.py:168-195), or the bf16 device tile."""
    if all(is_bf16(t) for t in io[0][:2] + io[1]):
        return plan_linear_bf16(io, config)
    return _ref_plan_linear(io, config)


MK.get_task_builder("linear").plan = _plan_linear_any
for _op, _fn in (("rmsnorm", plan_rmsnorm), ("attention", plan_attention),
                 ("allreduce_residual", plan_allreduce_residual)):
    if _op not in MK.registered_ops():
        MK.register_task_builder(_op, _fn)


# ---------------------------------------------------------------------- device tables
def layer_tables(program: MK.MegaProgram, built: MK.BuiltGraph):
    """Per-layer config rows and TMA map specs for tf_layer_megakernel_run."""
    cfg = np.zeros((max(len(built.layer_ops), 1), CFG_INTS), dtype=np.int32)
    specs: list = []

    def map_id(spec):
        if spec not in specs:
            specs.append(spec)
        return specs.index(spec)

    for lid, op in built.layer_ops.items():
        c = built.layer_configs[lid]
        ins, outs = program.layers[lid][1]
        if op not in LAYER_OP_CODES:
            raise BuildError(f"op {op!r} has no bf16 device implementation")
        row = cfg[lid]
        row[0] = LAYER_OP_CODES[op]
        row[3] = c.get("block_rows", 0)
        if op == "linear":
            x, w = ins[0], ins[1]
            m, k = x.shape
            n = w.shape[0]
            row[1], row[2] = BLOCK_M, BLOCK_N
            row[4] = EPILOGUES[c["epilogue"]]
            row[5] = map_id((x.offset, 2, k, m, 0, 64, 128, 0))
            row[6] = map_id((w.offset, 2, k, n, 0, 64, BLOCK_N, 0))
            if c["epilogue"] == "rope":
                row[9] = ins[2].shape[0]
                row[13] = c.get("rope_cols", n)
            row[14] = len(ins)  # io slot of the output
        elif op == "attention":
            (qkv,) = ins
            hq, hkv = c["heads_q"], c["heads_kv"]
            row[5] = map_id((qkv.offset, 3, HEAD_DIM, hq + 2 * hkv, qkv.shape[0], 64, 1, 128))
            row[7], row[8], row[9] = hq, hkv, c["seq_len"]
            row[10] = _f32_bits(c["scale"])
            row[12] = 1 if c["causal"] else 0
            row[14] = c["heads_per_task"]
        elif op == "rmsnorm":
            row[11] = _f32_bits(c["eps"])
        elif op == "allreduce_residual":
            row[13] = 1 if c.get("two_shot", True) else 0
            if c.get("norm_gain") is not None:
                row[11] = _f32_bits(c["eps"])
                row[15] = 1 + (c["norm_gain"].offset >> 4)
    for t in program.tensors:
        if t.offset % 16:
            raise BuildError(f"tensor {t.name} offset {t.offset} is not 16-byte aligned")
    spec_arr = np.array(specs, dtype=np.int64).reshape(-1, 8)
    return cfg, spec_arr


ELEMENTWISE_OPS = ("rmsnorm", "allreduce_residual")


def dataflow_order(built: MK.BuiltGraph, lag: int = 0) -> list:
    """Task order for the static queues: tensor tasks keep the builder's order;
    an elementwise task moves up to `lag` positions after the last producer tile it
    waits on (about two waves of round-robin queues, so its inputs are usually
    complete when its CTA reaches it), but never past its own builder position.
    Each CTA drains its queue in order, so an elementwise task queued behind the
    CTA's remaining GEMM tiles would wait for all of them (the final allreduce
    would trail the whole down-projection), while one queued too early blocks the
    CTA's epilogue warps.  An elementwise task only moves earlier and never ahead
    of its producers, so the result is a topological order and round-robin queues
    stay deadlock-free."""
    slot = {}
    keyed = []
    for i, t in enumerate(built.tasks):
        key = float(i)
        if built.layer_ops[t.layer_id] in ELEMENTWISE_OPS:
            deps = [slot.get((int(p), tile)) for p, lo, hi in built.dep_table[t.dep_start:t.dep_end]
                    for tile in range(int(lo), int(hi))]
            deps = [d for d in deps if d is not None]
            if deps:
                key = min(max(deps) + 0.5 + lag, float(i))
        slot[(t.task_id, t.tile_id)] = key
        keyed.append((key, i, t))
    keyed.sort(key=lambda x: (x[0], x[1]))
    return [t for _, _, t in keyed]


# per-SM rates for the static schedule's cost model (measured on B200, round 1):
# linear tiles ~9 TFLOP/s per SM (1.34 PFLOP/s sustained / 148), attention ~5.5,
# elementwise tasks are latency-bound at ~25 GB/s per CTA
_RATE_LINEAR, _RATE_ATTN, _RATE_ELEM = 9.0e12, 5.5e12, 25.0e9


def task_cost_us(built: MK.BuiltGraph, program: MK.MegaProgram, t) -> float:
    """Estimated duration of one task on one CTA (microseconds)."""
    op = built.layer_ops[t.layer_id]
    ins, outs = program.layers[t.layer_id][1]
    c = built.layer_configs[t.layer_id]
    if op == "linear":
        return 2.0 * BLOCK_M * BLOCK_N * ins[0].shape[1] / _RATE_LINEAR * 1e6
    if op == "attention":
        i = t.tile_id // (c["heads_q"] // c.get("heads_per_task", 1))  # tile = i * (hq / np) + hp
        tps = c["seq_len"] // 128
        n_kv = (i % tps) + 1 if c["causal"] else tps
        return 4.0 * 128 * 128 * HEAD_DIM * n_kv / _RATE_ATTN * 1e6 + 2.0
    rows = min(c["block_rows"], ins[0].shape[0] - t.tile_id * c["block_rows"])
    nbytes = rows * ins[0].shape[1] * 2 * (len(ins) + len(outs))
    return nbytes / _RATE_ELEM * 1e6 + 2.0


def list_schedule(program: MK.MegaProgram, built: MK.BuiltGraph, num_sms: int, order=None):
    """Static queues by simulated list scheduling: walk a topological task order and
    give each task to the CTA that can start it earliest (max of the CTA's free time
    and the task's inputs' estimated finish), appending it to that CTA's queue.
    Every queue is a subsequence of one topological order, so the in-order
    persistent executor cannot deadlock (the globally earliest unfinished task
    always has its inputs done and nothing ahead of it in its queue).  Balances the
    causal attention tiles (longest first), the GEMM waves and the elementwise
    tasks, which land on CTAs that run out of tensor work first."""
    import heapq
    order = list(built.tasks if order is None else order)
    finish = {}
    free = [(0.0, c) for c in range(num_sms)]
    heapq.heapify(free)
    queues = [[] for _ in range(num_sms)]
    for t in order:
        ready = 0.0
        for p, lo, hi in built.dep_table[t.dep_start:t.dep_end]:
            for tile in range(int(lo), int(hi)):
                f = finish.get((int(p), tile))
                if f is not None and f > ready:
                    ready = f
        # earliest-start CTA: the least-loaded one unless several are free before `ready`
        ft, cta = heapq.heappop(free)
        start = max(ft, ready)
        end = start + task_cost_us(built, program, t)
        finish[(t.task_id, t.tile_id)] = end
        queues[cta].append(t)
        heapq.heappush(free, (end, cta))
    slots = max(1, max(len(q) for q in queues))
    q = np.zeros((slots, num_sms, MK.INT_PER_TASK), dtype=np.int32)
    q[:, :, MK.IO_TENSORS_OFFSET::MK.INTS_PER_IO_SLOT] = -1
    counts = np.zeros(num_sms, dtype=np.int32)
    for c, tasks in enumerate(queues):
        for i, t in enumerate(tasks):
            q[i, c] = MK.encode_task(t)
        counts[c] = len(tasks)
    return q, counts


class LayerArgs(C.Structure):
    _fields_ = [("queues", C.c_void_p), ("counts", C.c_void_p), ("deps", C.c_void_p),
                ("layer_cfg", C.c_void_p), ("map_specs", C.c_void_p), ("num_maps", C.c_int32),
                ("num_sms", C.c_int32), ("max_tiles", C.c_int32), ("num_layers", C.c_int32),
                ("flag_base", C.c_uint64), ("epoch", C.c_uint64), ("timeout_ns", C.c_uint64),
                ("trace", C.c_void_p), ("trace_slots", C.c_int32)]


class LayerRunner:
    """Device state for repeated runs of one bf16 program: the team's symmetric
    heap holds every tensor at its declared offset (identical on all PEs),
    scoreboard flags are epoch-valued (run e waits for flags >= e, so no reset
    between runs), queues/deps/config live on the device.

    team=None: a local team whose PEs all share `device` (every rank
    co-scheduled in one launch, world * num_sms CTAs).  team=<IPC Team>: this
    process runs its own rank with num_sms CTAs; peers' heaps are IPC-mapped."""

    def __init__(self, program: MK.MegaProgram, built: MK.BuiltGraph | None = None, num_sms: int | None = None,
                 *, team=None, device: int = 0, queues=None, counts=None, timeout_s: float = 20.0,
                 schedule: str = "rr"):
        import torch

        from .shmem import SymmetricHeap, Team
        self.program = program
        self.built = built or program.build()
        world = program.topology.world_size
        self.world = world
        if team is None:
            nsm_dev = torch.cuda.get_device_properties(device).multi_processor_count
            num_sms = num_sms or nsm_dev // world
            team = Team(world, [device] * world, program._top + 4096,
                        (self.built.max_task_id + 1) * self.built.max_tiles_per_op + 64)
            self.rank = -1
            self.device = device
        else:
            if team.world != world:
                raise ValueError("team world size differs from the program topology")
            self.rank = team.rank if team.rank is not None else -1
            self.device = team.devices[team.rank] if team.rank is not None else team.devices[0]
            num_sms = num_sms or torch.cuda.get_device_properties(self.device).multi_processor_count
        self.team = team
        self.num_sms = int(num_sms)
        self.heap = SymmetricHeap(program.topology, team=team)
        self.handles = {}
        for t in program.tensors:
            h = self.heap.alloc(t.nbytes)
            if h.offset != t.offset:
                raise BuildError("heap layout must match the declared offsets (allocate the program's "
                                 "tensors first on a fresh team)")
            self.handles[t.name] = h
        nslots = (self.built.max_task_id + 1) * self.built.max_tiles_per_op
        self.flags = self.heap.alloc_signals(nslots)
        if queues is None:
            # "rr": the reference's round-robin over the builder order (fastest measured
            # at config 5: it keeps the GEMM waves' grouped raster); "dataflow" /
            # "list" are the alternatives measured in DESIGN.md §3.9
            if schedule == "rr":
                queues, counts = MK.encode_work_queues(self.built.tasks, self.num_sms)
            elif schedule == "dataflow":
                queues, counts = MK.encode_work_queues(dataflow_order(self.built, 2 * self.num_sms),
                                                       self.num_sms)
            elif schedule == "list":
                queues, counts = list_schedule(program, self.built, self.num_sms)
            else:
                raise ValueError(f"unknown schedule {schedule!r}")
        self.queues = np.ascontiguousarray(queues, dtype=np.int32)
        self.counts = np.ascontiguousarray(counts, dtype=np.int32)
        if self.queues.shape[1] != self.num_sms:
            raise ValueError("queues were encoded for a different SM count")
        cfg, specs = layer_tables(program, self.built)
        self.specs = np.ascontiguousarray(specs)
        dev = f"cuda:{self.device}"
        d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        self._tq, self._tc, self._tcfg = d(self.queues), d(self.counts), d(cfg)
        self._td = d(self.built.dep_table if self.built.dep_table.size else np.zeros((1, 3), np.int32))
        self.epoch = 0
        self.timeout_ns = int(timeout_s * 1e9)
        self.by_name = {t.name: t for t in program.tensors}

    def view(self, name: str, pe: int | None = None):
        """Torch view of tensor `name` in PE `pe`'s heap (bf16 tensors as torch.bfloat16)."""
        import torch
        t = self.by_name[name]
        pe = (self.rank if self.rank >= 0 else 0) if pe is None else pe
        dt = torch.bfloat16 if is_bf16(t) else np.dtype(t.dtype)
        return self.heap.view(self.handles[name], pe, dt, t.shape)

    def enable_trace(self, on: bool = True) -> None:
        """Per-task device timestamps (fetch, deps satisfied, released) for the next runs."""
        import torch
        ctas = self.num_sms * (self.world if self.rank < 0 else 1)
        self._trace = (torch.zeros(ctas, self.queues.shape[0], 4, dtype=torch.int64,
                                   device=f"cuda:{self.device}") if on else None)

    def trace(self):
        """[(cta, task_id, tile, t_fetch, t_deps_ok, t_done)] of the last traced run (ns)."""
        t = self._trace.cpu().numpy()
        out = []
        for cta in range(t.shape[0]):
            for idx in range(int(self.counts[cta % self.num_sms])):
                f, d, e, tt = (int(v) for v in t[cta, idx])
                if e:  # tasks a rank skips (two-shot allreduce tiles it does not own) leave no record
                    out.append((cta, tt >> 32, tt & 0xFFFFFFFF, f, d, e))
        return out

    def run(self, stream=None) -> None:
        import torch

        from . import _lib
        if not self.built.tasks:
            return
        self.epoch += 1
        tr = getattr(self, "_trace", None)
        args = LayerArgs(self._tq.data_ptr(), self._tc.data_ptr(), self._td.data_ptr(),
                         self._tcfg.data_ptr(), self.specs.ctypes.data, len(self.specs), self.num_sms,
                         self.built.max_tiles_per_op, len(self.built.layer_ops), self.flags.base,
                         self.epoch, self.timeout_ns, 0 if tr is None else tr.data_ptr(),
                         self.queues.shape[0])
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            if self.rank >= 0 and self.world > 1:
                # one launch per process: no rank may start writing peers' buffers (two-shot
                # allreduce) or its own partials (read by peers) while a peer still runs
                # the previous epoch -- stream-ordered team barrier first
                _lib.call("tf_barrier_all", self.team.handle, int(self.rank), s.cuda_stream)
            _lib.call("tf_layer_megakernel_run", self.team.handle, int(self.rank), C.byref(args),
                      s.cuda_stream)
            if self.rank >= 0 and self.world > 1:
                # two-shot allreduce tiles this rank does not own are P2P-stored into its
                # outputs by their owners; nothing in this launch waits for them, so close
                # the epoch with a second stream-ordered barrier: work enqueued after run()
                # on this stream sees every peer's rows
                _lib.call("tf_barrier_all", self.team.handle, int(self.rank), s.cuda_stream)

    def check(self) -> None:
        self.team.check()

    def close(self) -> None:
        self.team.close()


# ---------------------------------------------------------------------- Llama layer
def rope_table(seq_len: int, theta: float = 500000.0) -> np.ndarray:
    """[seq, 128] fp32: cos(pos * f_i) in [0, 64), sin in [64, 128), f_i = theta^(-2i/128)
    (Llama-3 rotate-half convention, pairs (i, i + 64) of each head)."""
    inv = theta ** (-np.arange(0, HEAD_DIM, 2, dtype=np.float64) / HEAD_DIM)
    ang = np.arange(seq_len, dtype=np.float64)[:, None] * inv[None, :]
    return np.concatenate([np.cos(ang), np.sin(ang)], axis=1).astype(np.float32)


def interleave_gate_up(w_gate: np.ndarray, w_up: np.ndarray, block: int = 128) -> np.ndarray:
    """[F, H] gate and up -> [2F, H] with 128-row blocks (gate_b, up_b) alternating, so
    one 128 x 256 output tile holds matching gate and up columns."""
    f = w_gate.shape[0]
    if f % block or w_up.shape != w_gate.shape:
        raise ValueError("gate/up must be [F, H] with F % 128 == 0")
    out = np.empty((2 * f, w_gate.shape[1]), dtype=w_gate.dtype)
    for b in range(f // block):
        out[2 * b * block:(2 * b + 1) * block] = w_gate[b * block:(b + 1) * block]
        out[(2 * b + 1) * block:(2 * b + 2) * block] = w_up[b * block:(b + 1) * block]
    return out


def llama_layer_program(topology, tokens: int, hidden: int, heads_q: int, heads_kv: int, ffn: int,
                        seq_len: int | None = None, eps: float = 1e-5, norm_rows: int = 8):
    """The TP-sharded Llama layer as a MegaProgram (per-rank shard shapes; TP =
    topology.world_size).  Returns (program, names)."""
    tp = topology.world_size
    if heads_q % tp or heads_kv % tp or ffn % tp:
        raise BuildError("heads and ffn must divide by the TP degree")
    hq, hkv, f = heads_q // tp, heads_kv // tp, ffn // tp
    seq = seq_len or tokens
    qkv_n = (hq + 2 * hkv) * HEAD_DIM
    p = MK.MegaProgram(topology)
    T = lambda name, shape, dt=bfloat16: p.tensor(name, shape, dt)
    x = T("x", (tokens, hidden))
    g1, g2 = T("g_attn", (1, hidden)), T("g_mlp", (1, hidden))
    rope = T("rope", (seq, HEAD_DIM), np.float32)
    wqkv = T("w_qkv", (qkv_n, hidden))
    wo = T("w_o", (hidden, hq * HEAD_DIM))
    w13 = T("w_gate_up", (2 * f, hidden))
    w2 = T("w_down", (hidden, f))
    xn, qkv = T("xn", (tokens, hidden)), T("qkv", (tokens, qkv_n))
    att, op = T("attn", (tokens, hq * HEAD_DIM)), T("o_part", (tokens, hidden))
    h, hn = T("h", (tokens, hidden)), T("hn", (tokens, hidden))
    act, dp = T("act", (tokens, f)), T("down_part", (tokens, hidden))
    out = T("out", (tokens, hidden))
    p.layer("rmsnorm", [x, g1], [xn], eps=eps, block_rows=norm_rows)
    p.layer("linear", [xn, wqkv, rope], [qkv], epilogue="rope", rope_cols=(hq + hkv) * HEAD_DIM)
    p.layer("attention", [qkv], [att], heads_q=hq, heads_kv=hkv, seq_len=seq, causal=True)
    p.layer("linear", [att, wo], [op])
    p.layer("allreduce_residual", [op, x], [h, hn], block_rows=norm_rows, norm_gain=g2, eps=eps)
    p.layer("linear", [hn, w13], [act], epilogue="silu_mul")
    p.layer("linear", [act, w2], [dp])
    p.layer("allreduce_residual", [dp, h], [out], block_rows=norm_rows)
    return p
