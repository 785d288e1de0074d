"""Task-level megakernel: task records, work queues, scoreboard, device executor.

Host side keeps the reference's wire contract bit-for-bit
(ovs/megakernel/encoding.py:20-204, builders.py:105-236, runner.py:45-118):
  * a task is INT_PER_TASK = 30 int32 words -- type, layer, task, tile,
    dependency-entry start/end, then 4 io slots of (byte offset, dtype tag,
    4 dims), offset -1 marking an empty slot;
  * queues are [slot][sm][INT_PER_TASK], tasks dealt round-robin over SMs;
  * dependency rows are (producer task, first tile, one-past-last tile) from
    region intersection; require_full inputs depend on every producer tile;
  * scoreboard slot = task_id * max_tiles_per_op + tile.

Device side (csrc/tf_mega.cu) is one persistent sm_100a kernel: every CTA
drains its queue, acquire-waits the dependency flags (on peers' scoreboards
for allreduce), runs the task -- linear = a tcgen05 kind::tf32 tile with an
fp32 TMEM accumulator, add = elementwise, allreduce = ascending-rank sum of
the peers' tiles read over P2P -- and release-stores its flag.  Tensors live
in the team's symmetric heap at the declared offsets; int64 ("exact mode")
inputs are stored as fp32 (exact for |x| < 2^24) and returned as int64.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from .errors import BuildError, ProtocolError

TASK_TYPE_OFFSET = 0
LAYER_ID_OFFSET = 1
TASK_ID_OFFSET = 2
TILE_ID_OR_START_OFFSET = 3
DEPEND_ENTRY_START_OFFSET = 4
DEPEND_ENTRY_END_OFFSET = 5
IO_TENSORS_OFFSET = 6
MAX_NUM_TENSOR_DIMS = 4
INTS_PER_IO_SLOT = 2 + MAX_NUM_TENSOR_DIMS
MAX_IO_TENSORS = 4
INT_PER_TASK = IO_TENSORS_OFFSET + MAX_IO_TENSORS * INTS_PER_IO_SLOT
INT_PER_DEPS = 3

DTYPE_TAGS = {np.dtype(np.float32): 0, np.dtype(np.int64): 1}
TAG_DTYPES = {v: k for k, v in DTYPE_TAGS.items()}
_INT32 = (-(2 ** 31), 2 ** 31 - 1)
OFFSET_SHIFT = 4


def _i32(v: int, what: str) -> int:
    if not _INT32[0] <= int(v) <= _INT32[1]:
        raise ValueError(f"{what}={v} does not fit an int32 word")
    return int(v)


@dataclass(frozen=True)
class IoSlot:
    offset: int
    dtype_tag: int
    dims: tuple

    @property
    def dtype(self):
        return TAG_DTYPES[self.dtype_tag]

    @property
    def nbytes(self) -> int:
        return int(np.prod(self.dims)) * self.dtype.itemsize


@dataclass(frozen=True)
class TaskRecord:
    task_type: int
    layer_id: int
    task_id: int
    tile_id: int
    dep_start: int
    dep_end: int
    io: tuple = ()


def encode_task(task: TaskRecord) -> np.ndarray:
    w = np.zeros(INT_PER_TASK, dtype=np.int32)
    for off, val, name in ((TASK_TYPE_OFFSET, task.task_type, "task_type"),
                           (LAYER_ID_OFFSET, task.layer_id, "layer_id"),
                           (TASK_ID_OFFSET, task.task_id, "task_id"),
                           (TILE_ID_OR_START_OFFSET, task.tile_id, "tile_id"),
                           (DEPEND_ENTRY_START_OFFSET, task.dep_start, "dep_start"),
                           (DEPEND_ENTRY_END_OFFSET, task.dep_end, "dep_end")):
        w[off] = _i32(val, name)
    if len(task.io) > MAX_IO_TENSORS:
        raise ValueError(f"at most {MAX_IO_TENSORS} io tensors per task")
    for i in range(MAX_IO_TENSORS):
        base = IO_TENSORS_OFFSET + i * INTS_PER_IO_SLOT
        if i >= len(task.io):
            w[base] = -1
            continue
        slot = task.io[i]
        if not 1 <= len(slot.dims) <= MAX_NUM_TENSOR_DIMS or min(slot.dims) < 1:
            raise ValueError(f"io tensor needs 1..{MAX_NUM_TENSOR_DIMS} dims >= 1, got {slot.dims}")
        off, tag = slot.offset, slot.dtype_tag
        if off > _INT32[1] and off % 16 == 0:
            # extension for heaps past 2 GiB (the reference's are < 2 GiB, where the
            # encoding is unchanged): offset in 16-byte units, shift in tag bits 8-11
            off, tag = off >> OFFSET_SHIFT, tag | (OFFSET_SHIFT << 8)
        w[base] = _i32(off, "io offset")
        w[base + 1] = _i32(tag, "dtype tag")
        w[base + 2:base + 2 + len(slot.dims)] = [_i32(d, "dim") for d in slot.dims]
    return w


def decode_task(words) -> TaskRecord:
    words = np.asarray(words)
    io = []
    for i in range(MAX_IO_TENSORS):
        base = IO_TENSORS_OFFSET + i * INTS_PER_IO_SLOT
        if int(words[base]) < 0:
            continue
        dims = tuple(int(d) for d in words[base + 2:base + 2 + MAX_NUM_TENSOR_DIMS] if d != 0)
        tag = int(words[base + 1])
        io.append(IoSlot(int(words[base]) << ((tag >> 8) & 0xF), tag & 0xFF, dims))
    return TaskRecord(*(int(words[o]) for o in range(IO_TENSORS_OFFSET)), io=tuple(io))


def encode_work_queues(tasks, num_sms: int):
    """Round-robin over num_sms queues -> (int32 [slots, num_sms, INT_PER_TASK], counts)."""
    if num_sms < 1:
        raise ValueError("num_sms must be >= 1")
    slots = max(1, -(-len(tasks) // num_sms))
    q = np.zeros((slots, num_sms, INT_PER_TASK), dtype=np.int32)
    q[:, :, IO_TENSORS_OFFSET::INTS_PER_IO_SLOT] = -1
    counts = np.zeros(num_sms, dtype=np.int32)
    for i, t in enumerate(tasks):
        q[i // num_sms, i % num_sms] = encode_task(t)
        counts[i % num_sms] += 1
    return q, counts


def fetch_task(queues, idx: int, sm_id: int, counts=None, runtime_scheduler: bool = False):
    """Decode entry (idx, sm_id) with the device's flat address arithmetic."""
    flat = np.asarray(queues).reshape(-1)
    if runtime_scheduler:
        if not 0 <= idx < flat.size // INT_PER_TASK:
            raise ValueError(f"queue index {idx} out of range")
        return decode_task(flat[idx * INT_PER_TASK:(idx + 1) * INT_PER_TASK])
    slots, nsm, _ = np.asarray(queues).shape
    if counts is not None and not 0 <= idx < int(counts[sm_id]):
        raise ValueError(f"queue index {idx} out of range for sm {sm_id}")
    if not (0 <= idx < slots and 0 <= sm_id < nsm):
        raise ValueError(f"queue index ({idx}, {sm_id}) out of range")
    base = (idx * nsm + sm_id) * INT_PER_TASK
    return decode_task(flat[base:base + INT_PER_TASK])


def queues_to_bytes(q) -> bytes:
    return np.ascontiguousarray(q, dtype="<i4").tobytes()


def queues_from_bytes(buf: bytes, num_sms: int):
    w = np.frombuffer(buf, dtype="<i4")
    if w.size % (num_sms * INT_PER_TASK):
        raise ValueError("work-queue byte length inconsistent with layout")
    return w.reshape(-1, num_sms, INT_PER_TASK).copy()


def deps_to_bytes(d) -> bytes:
    return np.ascontiguousarray(d, dtype="<i4").tobytes()


def deps_from_bytes(buf: bytes):
    w = np.frombuffer(buf, dtype="<i4")
    if w.size % INT_PER_DEPS:
        raise ValueError("dependency table byte length inconsistent with layout")
    return w.reshape(-1, INT_PER_DEPS).copy()


def dump_task_graph(tasks, dep_table) -> str:
    out = []
    for t in tasks:
        deps = [f"task {int(r[0])} tiles [{int(r[1])},{int(r[2])})"
                for r in dep_table[t.dep_start:t.dep_end]]
        out.append(f"task {t.task_id}:{t.tile_id}" + (" <- " + "; ".join(deps) if deps else ""))
    return "\n".join(out)


# ---------------------------------------------------------------------- builders
@dataclass(frozen=True)
class MkTensor:
    name: str
    offset: int
    dtype: np.dtype
    shape: tuple

    @property
    def nbytes(self) -> int:
        return int(np.prod(self.shape)) * np.dtype(self.dtype).itemsize

    def io_slot(self) -> IoSlot:
        return IoSlot(self.offset, DTYPE_TAGS[np.dtype(self.dtype)], tuple(int(d) for d in self.shape))


@dataclass(frozen=True)
class InputDependencyDesc:
    tensor: MkTensor
    require_full: bool = False
    start_indices: tuple = (0, 0)
    data_sizes: tuple | None = None


@dataclass(frozen=True)
class OutputTilingDesc:
    tile_sizes: tuple


@dataclass(frozen=True)
class TileSpec:
    tile_id: int
    inputs: tuple


@dataclass
class LayerPlan:
    op_type: str
    io_tensors: list
    config: dict
    num_tiles: int
    tiles: list
    out_tiling: dict


@dataclass
class Builder:
    op_type: str
    task_type: int
    plan: Callable


_REGISTRY: dict = {}


def register_task_builder(op_type: str, plan_fn) -> None:
    if op_type in _REGISTRY:
        raise ProtocolError(f"op_type {op_type!r} already registered")
    _REGISTRY[op_type] = Builder(op_type, len(_REGISTRY), plan_fn)


def get_task_builder(op_type: str) -> Builder:
    if op_type not in _REGISTRY:
        raise BuildError(f"unknown op_type {op_type!r}; registered: {list(_REGISTRY)}")
    return _REGISTRY[op_type]


def registered_ops() -> list:
    return list(_REGISTRY)


@dataclass
class BuiltGraph:
    tasks: list
    dep_table: np.ndarray
    layer_configs: dict
    layer_ops: dict
    max_task_id: int
    max_tiles_per_op: int


def _tile_ranges(desc: InputDependencyDesc, tiling: OutputTilingDesc, tensor: MkTensor):
    """Producer tile-id ranges [lo, hi) intersecting the input region."""
    r0, c0 = desc.start_indices
    sz = desc.data_sizes or tensor.shape
    r1, c1 = r0 + sz[0], c0 + sz[1]
    rows, cols = tensor.shape
    if r0 < 0 or c0 < 0 or r1 > rows or c1 > cols:
        raise BuildError(f"input region [{r0}:{r1}, {c0}:{c1}] exceeds {tensor.name} of shape {tensor.shape}")
    tm_, tn_ = tiling.tile_sizes
    per_row = -(-cols // tn_)
    for tm in range(r0 // tm_, (r1 - 1) // tm_ + 1):
        yield tm * per_row + c0 // tn_, tm * per_row + (c1 - 1) // tn_ + 1


def build_task_graph(layers, device_prop=None) -> BuiltGraph:
    """One task record per tile of every layer plus the dependency table."""
    producers, tasks, deps, cfgs, ops = {}, [], [], {}, {}
    max_tiles = 1
    for layer_id, (op_type, io_tensors, config) in enumerate(layers):
        b = get_task_builder(op_type)
        plan = b.plan(io_tensors, dict(config))
        cfgs[layer_id], ops[layer_id] = plan.config, op_type
        max_tiles = max(max_tiles, plan.num_tiles)
        slots = tuple(t.io_slot() for t in io_tensors[0] + io_tensors[1])
        for tile in plan.tiles:
            start = len(deps)
            for d in tile.inputs:
                prod = producers.get(d.tensor.name)
                if prod is None:
                    continue
                p_task, p_tiling, p_tensor, p_tiles = prod
                if d.require_full:
                    deps.append((p_task, 0, p_tiles))
                else:
                    deps.extend((p_task, lo, hi) for lo, hi in _tile_ranges(d, p_tiling, p_tensor))
            tasks.append(TaskRecord(b.task_type, layer_id, layer_id, tile.tile_id, start, len(deps), slots))
        for out in io_tensors[1]:
            producers[out.name] = (layer_id, plan.out_tiling[out.name], out, plan.num_tiles)
    table = np.array(deps, dtype=np.int32).reshape(-1, INT_PER_DEPS)
    return BuiltGraph(tasks, table, cfgs, ops, len(layers) - 1 if layers else 0, max_tiles)


def _plan_linear(io, config) -> LayerPlan:
    (x, w), (y,) = io[0], io[1]
    m, k = x.shape
    n, wk = w.shape
    if wk != k or y.shape != (m, n):
        raise BuildError(f"linear shapes inconsistent: x{x.shape} w{w.shape} y{y.shape}")
    cfg = {"block_m": 16, "block_n": 16, "block_k": 16, "num_stages": 3, **config}
    bm, bn = cfg["block_m"], cfg["block_n"]
    tm_n, tn_n = -(-m // bm), -(-n // bn)
    tiles = [TileSpec(tm * tn_n + tn, (
        InputDependencyDesc(x, start_indices=(tm * bm, 0), data_sizes=(min(bm, m - tm * bm), k)),
        InputDependencyDesc(w, start_indices=(tn * bn, 0), data_sizes=(min(bn, n - tn * bn), k))))
        for tm in range(tm_n) for tn in range(tn_n)]
    return LayerPlan("linear", io, cfg, tm_n * tn_n, tiles, {y.name: OutputTilingDesc((bm, bn))})


def _plan_rows(op, io, config, full_input):
    ins, (y,) = io[0], io[1]
    if any(t.shape != y.shape for t in ins):
        raise BuildError(f"{op} shapes must match: {[t.shape for t in ins]} {y.shape}")
    cfg = {"block_rows": 16, **config}
    rows, cols = y.shape
    br = cfg["block_rows"]
    n = -(-rows // br)
    tiles = []
    for tm in range(n):
        if full_input:
            inputs = tuple(InputDependencyDesc(t, require_full=True) for t in ins)
        else:
            reg = dict(start_indices=(tm * br, 0), data_sizes=(min(br, rows - tm * br), cols))
            inputs = tuple(InputDependencyDesc(t, **reg) for t in ins)
        tiles.append(TileSpec(tm, inputs))
    return LayerPlan(op, io, cfg, n, tiles, {y.name: OutputTilingDesc((br, cols))})


register_task_builder("linear", _plan_linear)
register_task_builder("add", lambda io, cfg: _plan_rows("add", io, cfg, False))
register_task_builder("allreduce", lambda io, cfg: _plan_rows("allreduce", io, cfg, True))


@dataclass(frozen=True)
class DeviceProp:
    """Persistent CTAs per rank the executor may use (runner.py:27-29)."""
    num_sms: int


@dataclass
class MegaProgram:
    """Heap tensors (16-byte bump offsets) and layers (runner.py:45-60)."""

    topology: object
    tensors: list = field(default_factory=list)
    layers: list = field(default_factory=list)
    _top: int = 0

    def tensor(self, name: str, shape, dtype) -> MkTensor:
        if any(t.name == name for t in self.tensors):
            raise BuildError(f"tensor {name!r} already declared")
        off = -(-self._top // 16) * 16
        t = MkTensor(name, off, np.dtype(dtype), tuple(int(d) for d in shape))
        self._top = off + t.nbytes
        self.tensors.append(t)
        return t

    def layer(self, op_type: str, inputs, outputs, **config) -> None:
        get_task_builder(op_type)
        self.layers.append((op_type, [list(inputs), list(outputs)], config))

    def build(self, device_prop=None) -> BuiltGraph:
        return build_task_graph(self.layers, device_prop)


# ---------------------------------------------------------------------- device run
@dataclass
class MegaRun:
    outputs: dict
    trace: object
    heap: object
    scoreboards: list


class Scoreboard:
    """Host view of one rank's scoreboard flags (scoreboard.py:19-59)."""

    def __init__(self, heap, flags, dep_table, max_task_id, max_tiles_per_op, rank):
        self.heap, self.flags, self.dep_table = heap, flags, dep_table
        self.max_task_id, self.max_tiles_per_op, self.rank = max_task_id, max_tiles_per_op, rank

    def _slot(self, task_id: int, tile: int) -> int:
        return task_id * self.max_tiles_per_op + tile

    def flags_view(self, pe: int) -> np.ndarray:
        return self.heap.sig_view(self.flags, pe)


class MegaArgs(C.Structure):
    _fields_ = [("queues", C.c_void_p), ("counts", C.c_void_p), ("deps", C.c_void_p),
                ("task_ops", C.c_void_p), ("layer_cfg", C.c_void_p), ("num_sms", C.c_int32),
                ("slots", C.c_int32), ("max_tiles", C.c_int32), ("num_layers", C.c_int32),
                ("flag_base", C.c_uint64), ("epoch", C.c_uint64), ("timeout_ns", C.c_uint64)]


OP_CODES = {"linear": 0, "add": 1, "allreduce": 2}


def run_megakernel(program: MegaProgram, built: BuiltGraph, num_sms: int, *, queues=None, counts=None,
                   inputs: dict | None = None, seed: int = 0, debug_scoreboard: bool = True,
                   devices=None, timeout_s: float = 20.0) -> MegaRun:
    """Execute the task graph on every rank with num_sms persistent CTAs per rank."""
    import torch

    from . import _lib
    from .shmem import SymmetricHeap, Team

    topo = program.topology
    world = topo.world_size
    if num_sms < 1 or num_sms > topo.num_sms:
        raise ValueError(f"num_sms must be in [1, {topo.num_sms}]")
    if any(_layer.is_bf16(t) for t in program.tensors):
        return _run_bf16(program, built, num_sms, queues, counts, inputs or {}, devices, timeout_s)
    if queues is None:
        queues, counts = encode_work_queues(built.tasks, num_sms)
    elif counts is None:
        raise ValueError("explicit queues need explicit counts")
    queues = np.ascontiguousarray(queues, dtype=np.int32)
    counts = np.ascontiguousarray(counts, dtype=np.int32)
    if queues.shape[1] != num_sms:
        raise ValueError("queues were encoded for a different SM count")
    for t in program.tensors:
        if len(t.shape) != 2:
            raise BuildError("device megakernel tensors are 2-D")
    if devices is None:
        ndev = torch.cuda.device_count()
        if ndev == 0:
            raise RuntimeError("no CUDA device: the megakernel has no CPU path")
        devices = [0] * world  # all ranks co-resident in one launch on one GPU
    if len(set(devices)) != 1:
        raise ValueError("the single-process megakernel co-schedules all ranks on one device")
    nslots = (built.max_task_id + 1) * built.max_tiles_per_op
    # fp32 storage for both dtypes (int64 inputs exact below 2^24)
    heap_bytes = program._top * 2 + 4096  # int64 tensors shrink to fp32; keep offsets
    team = Team(world, devices, max(heap_bytes, 1 << 16), nslots + 64)
    heap = SymmetricHeap(topo, team=team)
    for t in program.tensors:  # identical bump layout (runner.py:85-87)
        h = heap.alloc(t.nbytes)
        if h.offset != t.offset:
            raise ProtocolError("heap layout must match the declared offsets")
    flags = heap.alloc_signals(nslots)
    inputs = inputs or {}
    by_name = {t.name: t for t in program.tensors}
    dev = devices[0]
    for name, value in inputs.items():
        t = by_name[name]
        per_rank = value if isinstance(value, (list, tuple)) else [value] * world
        if len(per_rank) != world:
            raise ValueError(f"input {name!r} needs {world} per-rank arrays")
        for r, arr in enumerate(per_rank):
            a = np.asarray(arr).reshape(t.shape).astype(np.float32)
            dst = heap.view(_handle(t), r, np.float32, t.shape)
            dst.copy_(torch.from_numpy(a).to(dst.device))
    # per-layer config table: [op, block_m, block_n, block_rows]
    cfg = np.zeros((max(len(built.layer_ops), 1), 4), dtype=np.int32)
    for lid, op in built.layer_ops.items():
        c = built.layer_configs[lid]
        cfg[lid] = [OP_CODES[op], c.get("block_m", 0), c.get("block_n", 0), c.get("block_rows", 0)]
        if op == "linear" and (c["block_m"] > 128 or c["block_n"] > 256):
            raise BuildError("device linear tiles need block_m <= 128 and block_n <= 256")
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(f"cuda:{dev}")
    tq, tc = d(queues), d(counts)
    tdeps = d(built.dep_table if built.dep_table.size else np.zeros((1, 3), np.int32))
    tcfg = d(cfg)
    args = MegaArgs(tq.data_ptr(), tc.data_ptr(), tdeps.data_ptr(), 0, tcfg.data_ptr(), num_sms,
                    queues.shape[0], built.max_tiles_per_op, len(built.layer_ops), flags.base, 1,
                    int(timeout_s * 1e9))
    torch.cuda.synchronize(dev)
    if built.tasks:
        with torch.cuda.device(dev):
            _lib.call("tf_megakernel_run", team.handle, C.byref(args),
                      torch.cuda.current_stream(dev).cuda_stream)
    torch.cuda.synchronize(dev)
    team.check()
    outputs = {}
    for t in program.tensors:
        vals = [heap.view(_handle(t), r, np.float32, t.shape).cpu().numpy() for r in range(world)]
        if np.dtype(t.dtype) == np.int64:
            vals = [np.rint(v).astype(np.int64) for v in vals]
        outputs[t.name] = vals
    boards = [Scoreboard(heap, flags, built.dep_table, built.max_task_id, built.max_tiles_per_op, r)
              for r in range(world)]
    return MegaRun(outputs, None, heap, boards)


def _handle(t: MkTensor):
    from .shmem import SymmHandle
    return SymmHandle(offset=t.offset, nbytes=t.nbytes)


def _run_bf16(program, built, num_sms, queues, counts, inputs, devices, timeout_s) -> MegaRun:
    """bf16 programs (transformer-layer ops) run on the fused-layer kernel."""
    import torch
    if torch.cuda.device_count() == 0:
        raise RuntimeError("no CUDA device: the megakernel has no CPU path")
    world = program.topology.world_size
    dev = 0 if devices is None else devices[0]
    if devices is not None and len(set(devices)) != 1:
        raise ValueError("the single-process megakernel co-schedules all ranks on one device")
    if queues is not None and counts is None:
        raise ValueError("explicit queues need explicit counts")
    runner = _layer.LayerRunner(program, built, num_sms, device=dev, queues=queues, counts=counts,
                                timeout_s=timeout_s)
    for name, value in inputs.items():
        t = runner.by_name[name]
        per_rank = value if isinstance(value, (list, tuple)) else [value] * world
        if len(per_rank) != world:
            raise ValueError(f"input {name!r} needs {world} per-rank arrays")
        for r, arr in enumerate(per_rank):
            v = runner.view(name, r)
            src = torch.as_tensor(np.asarray(arr, dtype=np.float32).reshape(t.shape))
            v.copy_(src.to(v.dtype).to(v.device))
    torch.cuda.synchronize(dev)
    runner.run()
    torch.cuda.synchronize(dev)
    runner.check()
    outputs = {t.name: [runner.view(t.name, r).float().cpu().numpy() for r in range(world)]
               for t in program.tensors}
    boards = [Scoreboard(runner.heap, runner.flags, runner.built.dep_table, runner.built.max_task_id,
                         runner.built.max_tiles_per_op, r) for r in range(world)]
    return MegaRun(outputs, None, runner.heap, boards)


from . import layer as _layer  # noqa: E402  (registers the bf16 layer ops)
