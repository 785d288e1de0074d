"""Device symmetric heap: the B200 replacement of ovs/shmem.py:87-473.

`SymmetricHeap` keeps the reference's host-visible API -- alloc /
alloc_collective / alloc_signals / view / sig_view / symm_at / remote_ptr and
the one-sided data and signal ops -- on top of a C-ABI team (libtilefuse).
Every PE's region is real device memory; `view()` returns a zero-copy torch
tensor of it, `sig_view()` a host snapshot of the uint64 signal slots.

The reference's generator-style device ops (`yield from heap.wait(...)`) have
no host meaning on hardware: the device side of those primitives lives in
csrc/tf_ptx.cuh (ld.acquire.sys / st.release.sys / red.release.sys spins used
inside the kernels).  The host methods here enqueue the same semantics on CUDA
streams: putmem/getmem are copy-engine transfers, putmem_signal orders the
signal after the payload, wait blocks the stream until all slots reach the
value, barrier_all is a stream-ordered all-rank rendezvous.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ProtocolError
from .topology import Topology

SCOPES = ("gpu", "sys")
SEMANTICS = ("relaxed", "acquire", "release")


@dataclass(frozen=True)
class SymmHandle:
    offset: int
    nbytes: int
    space: str = "heap"  # "heap" (P2P symmetric heap) or "nvls" (multicast region)


@dataclass(frozen=True)
class SigHandle:
    base: int
    nslots: int


@dataclass(frozen=True)
class Token:
    """Ordering witness returned by wait() (shmem.py:46-52).  On the device the wait
    is stream-ordered, so the token only records what was waited for."""
    pe: int
    slot: int
    num_slots: int
    time: float = 0.0


def consume_token(value, token: Token):
    """Returns `value` unchanged (shmem.py:55-57)."""
    return value


class _CudaMem:
    """Minimal __cuda_array_interface__ exporter for zero-copy torch views."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {
            "shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
            "version": 3, "strides": None,
        }


def tensor_from_ptr(ptr: int, nbytes: int, device: int) -> torch.Tensor:
    with torch.cuda.device(device):
        return torch.as_tensor(_CudaMem(ptr, nbytes), device=f"cuda:{device}")


def _stream_ptr(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


@dataclass(frozen=True)
class RemoteRegion:
    """Addressable view of one PE's copy of a symmetric region (shmem.py:65-77)."""

    heap: "SymmetricHeap"
    handle: SymmHandle
    pe: int

    @property
    def nbytes(self) -> int:
        return self.handle.nbytes

    def view(self, dtype, shape=None, offset: int = 0):
        return self.heap.view(self.handle, self.pe, dtype, shape=shape, offset=offset)


HANDLE_BLOB = 128


def share_fd(fd: int | None, group=None) -> int:
    """Pass rank 0's file descriptor to every rank of the group (SCM_RIGHTS over an
    abstract Unix socket whose name travels through torch.distributed).  Rank 0
    returns its own fd; the others a duplicate they own.  Used for the NVLS
    multicast handle (POSIX fd export, tf_team_nvls_create)."""
    import os
    import socket
    import uuid

    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    name = [f"\0tilefuse-fd-{os.getpid()}-{uuid.uuid4().hex}" if rank == 0 else None]
    dist.broadcast_object_list(name, src=0, group=group)
    if world == 1:
        return fd
    if rank == 0:
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(name[0])
        srv.listen(world)
        dist.barrier(group)
        try:
            for _ in range(world - 1):
                conn, _ = srv.accept()
                with conn:
                    socket.send_fds(conn, [b"fd"], [int(fd)])
        finally:
            srv.close()
        dist.barrier(group)
        return fd
    dist.barrier(group)
    with socket.socket(socket.AF_UNIX, socket.SOCK_STREAM) as c:
        c.connect(name[0])
        _, fds, _, _ = socket.recv_fds(c, 16, 1)
    dist.barrier(group)
    if len(fds) != 1:
        raise ProtocolError("file descriptor transfer failed")
    return fds[0]


def exchange_handles(blob: bytes, group=None) -> bytes:
    """All-gather one fixed-size IPC handle blob per rank over torch.distributed;
    returns the concatenation in rank order (what tf_team_open_peers expects).
    Works on any backend (gloo in the CPU tests, nccl on the GPU box)."""
    import torch.distributed as dist
    if len(blob) != HANDLE_BLOB:
        raise ValueError(f"handle blob must be {HANDLE_BLOB} bytes")
    world = dist.get_world_size(group)
    gathered = [None] * world
    dist.all_gather_object(gathered, blob, group=group)
    for b in gathered:
        if not isinstance(b, bytes) or len(b) != HANDLE_BLOB:
            raise ProtocolError("mismatched handle blobs in team creation")
    return b"".join(gathered)


class Team:
    """Owns a C tf_team.  Local (all PEs in this process) or IPC (one PE here)."""

    def __init__(self, world: int, devices=None, heap_bytes: int = 1 << 24,
                 signal_slots: int = 1 << 14, *, ipc_rank: int | None = None,
                 ipc_device: int | None = None):
        self.world = int(world)
        self.heap_bytes = int(heap_bytes)
        self.signal_slots = int(signal_slots)
        h = C.c_void_p()
        if ipc_rank is None:
            if devices is None:
                ndev = torch.cuda.device_count()
                devices = [r % max(ndev, 1) if ndev >= world else 0 for r in range(world)]
            self.devices = [int(d) for d in devices]
            arr = (C.c_int * self.world)(*self.devices)
            _lib.call("tf_team_create_local", self.world, arr, self.heap_bytes,
                      self.signal_slots, C.byref(h))
            self.rank = None
        else:
            dev = torch.cuda.current_device() if ipc_device is None else int(ipc_device)
            self.devices = [dev] * self.world
            _lib.call("tf_team_create_ipc", self.world, int(ipc_rank), dev, self.heap_bytes,
                      self.signal_slots, C.byref(h))
            self.rank = int(ipc_rank)
        self.handle = h

    @classmethod
    def from_process_group(cls, heap_bytes: int, signal_slots: int = 1 << 14, group=None,
                           nvls_bytes: int = 0):
        """IPC team over the current torch.distributed group (one GPU per rank).
        nvls_bytes > 0 also tries to create the NVLS multicast region (enable_nvls)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        team = cls(world, heap_bytes=heap_bytes, signal_slots=signal_slots, ipc_rank=rank,
                   ipc_device=torch.cuda.current_device())
        blob = (C.c_uint8 * HANDLE_BLOB)()
        _lib.call("tf_team_export_handle", team.handle, blob, HANDLE_BLOB)
        allb = exchange_handles(bytes(blob), group)
        _lib.call("tf_team_open_peers", team.handle, C.c_char_p(allb), HANDLE_BLOB)
        if nvls_bytes > 0:
            team.enable_nvls(nvls_bytes, group)
        return team

    # ------------------------------------------------------------------ NVLS
    @staticmethod
    def nvls_supported(device: int) -> bool:
        ok = C.c_int()
        _lib.call("tf_nvls_supported", int(device), C.byref(ok))
        return bool(ok.value)

    def enable_nvls(self, nbytes: int, group=None) -> bool:
        """Create the team's NVLS multicast region (multimem_ld_reduce / multimem_st
        in the switch, tf_nvls.cu).  Returns False -- and the team keeps its P2P
        paths -- when the devices do not support multicast or the driver refuses
        the object (e.g. a single-GPU lease).  IPC teams call it on every rank."""
        if self.rank is None:
            if not self.distinct_devices or self.world < 2:
                return False
            fd = C.c_int(-1)
            rc = _lib.lib().tf_team_nvls_create(self.handle, int(nbytes), C.byref(fd))
            return rc == 0
        import os

        import torch.distributed as dist
        ok = [None] * self.world
        dist.all_gather_object(ok, self.nvls_supported(self.devices[self.rank]) and self.world > 1,
                               group=group)
        if not all(ok):
            return False
        fd = C.c_int(-1)
        status = [0]
        if self.rank == 0:
            status[0] = _lib.lib().tf_team_nvls_create(self.handle, int(nbytes), C.byref(fd))
        dist.broadcast_object_list(status, src=0, group=group)
        if status[0] != 0:
            return False
        got = share_fd(fd.value if self.rank == 0 else None, group)
        rc = 0
        if self.rank != 0:
            rc = _lib.lib().tf_team_nvls_import(self.handle, int(nbytes), int(got))
            os.close(got)
        rc = rc or _lib.lib().tf_team_nvls_add_device(self.handle)
        rcs = [None] * self.world
        dist.all_gather_object(rcs, rc, group=group)
        if any(rcs):
            return False
        _lib.call("tf_team_nvls_bind", self.handle)
        dist.barrier(group)
        if self.rank == 0:
            os.close(fd.value)
        return True

    @property
    def nvls_enabled(self) -> bool:
        en = C.c_int()
        _lib.call("tf_nvls_enabled", self.handle, C.byref(en), None)
        return bool(en.value)

    def nvls_ptr(self, pe: int, offset: int) -> tuple[int, int]:
        uc, mc = C.c_void_p(), C.c_void_p()
        _lib.call("tf_nvls_ptr", self.handle, int(pe), int(offset), C.byref(uc), C.byref(mc))
        return int(uc.value or 0), int(mc.value or 0)

    @property
    def distinct_devices(self) -> bool:
        return len(set(self.devices)) == len(self.devices)

    def local_ranks(self):
        return [self.rank] if self.rank is not None else list(range(self.world))

    def check(self):
        _lib.call("tf_team_check", self.handle)

    def close(self):
        if self.handle:
            _lib.lib().tf_team_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def heap_ptr(self, pe: int, offset: int) -> int:
        p = C.c_void_p()
        _lib.call("tf_heap_ptr", self.handle, int(pe), int(offset), C.byref(p))
        return int(p.value or 0)

    def signal_ptr(self, pe: int, slot: int) -> int:
        p = C.c_void_p()
        _lib.call("tf_signal_ptr", self.handle, int(pe), int(slot), C.byref(p))
        return int(p.value or 0)


class SymmetricHeap:
    """Per-PE mirrored device regions plus uint64 signal slots (shmem.py:87-105).

    `topology` fixes the world size; `devices` maps PEs to CUDA devices (defaults
    to one GPU per PE when enough exist, else every PE on cuda:0).  The `engine`
    argument of the reference constructor is accepted and ignored.
    """

    def __init__(self, topology: Topology, engine=None, data_bytes: int = 1 << 24,
                 signal_slots: int = 1 << 14, *, devices=None, team: Team | None = None):
        self.topology = topology
        self.engine = engine
        self.data_bytes = int(data_bytes)
        self.signal_slots = int(signal_slots)
        self.team = team or Team(topology.world_size, devices, self.data_bytes, self.signal_slots)

    # ------------------------------------------------------------------ alloc
    def alloc(self, nbytes: int, align: int = 16) -> SymmHandle:
        if nbytes < 0:
            raise ValueError("allocation size must be >= 0")
        off = C.c_uint64()
        _lib.call("tf_heap_alloc", self.team.handle, int(nbytes), int(align), C.byref(off))
        return SymmHandle(offset=int(off.value), nbytes=int(nbytes))

    def alloc_collective(self, sizes) -> SymmHandle:
        sizes = list(sizes)
        if len(sizes) != self.topology.world_size:
            raise ProtocolError(f"collective allocation needs {self.topology.world_size} "
                                f"requests, got {len(sizes)}")
        if len(set(sizes)) != 1:
            raise ProtocolError(f"mismatched collective allocation sizes: {sizes}")
        return self.alloc(sizes[0])

    def alloc_multimem(self, nbytes: int, align: int = 16) -> SymmHandle:
        """Symmetric allocation in the team's NVLS multicast region (Team.enable_nvls):
        multimem_ld_reduce / multimem_st on it run as multimem instructions reduced
        and replicated in the NVSwitch.  Falls back to the P2P heap when NVLS is off."""
        if nbytes < 0:
            raise ValueError("allocation size must be >= 0")
        if not self.team.nvls_enabled:
            return self.alloc(nbytes, max(align, 16))
        off = C.c_uint64()
        _lib.call("tf_nvls_alloc", self.team.handle, int(nbytes), int(align), C.byref(off))
        return SymmHandle(offset=int(off.value), nbytes=int(nbytes), space="nvls")

    def alloc_signals(self, nslots: int) -> SigHandle:
        if nslots < 0:
            raise ValueError("signal slot count must be >= 0")
        base = C.c_uint64()
        _lib.call("tf_signal_alloc", self.team.handle, int(nslots), C.byref(base))
        return SigHandle(base=int(base.value), nslots=int(nslots))

    # ------------------------------------------------------------------ views
    def _check_pe(self, pe: int):
        if not 0 <= pe < self.topology.world_size:
            raise ValueError(f"pe {pe} out of range [0, {self.topology.world_size})")

    def view(self, handle: SymmHandle, pe: int, dtype, shape=None, offset: int = 0):
        """Zero-copy torch view of PE `pe`'s copy (shmem.py:143-153)."""
        self._check_pe(pe)
        if offset < 0 or offset > handle.nbytes:
            raise ValueError(f"offset {offset} outside region of {handle.nbytes} bytes")
        nbytes = handle.nbytes - offset
        tdtype = _torch_dtype(dtype)
        dev = self.team.devices[pe] if self.team.rank is None else self.team.devices[self.team.rank]
        if nbytes == 0:
            raw = torch.empty(0, dtype=torch.uint8, device=f"cuda:{dev}")
        elif handle.space == "nvls":
            raw = tensor_from_ptr(self.team.nvls_ptr(pe, handle.offset + offset)[0], nbytes, dev)
        else:
            raw = tensor_from_ptr(self.team.heap_ptr(pe, handle.offset + offset), nbytes, dev)
        isz = torch.empty(0, dtype=tdtype).element_size()
        arr = raw[: (nbytes // isz) * isz].view(tdtype)
        if shape is not None:
            count = int(np.prod(shape)) if shape else 1
            arr = arr[:count].reshape(shape)
        return arr

    def sig_view(self, sig: SigHandle, pe: int) -> np.ndarray:
        """Host snapshot of the signal slots (shmem.py:155-157), int64 like the reference."""
        self._check_pe(pe)
        out = (C.c_uint64 * max(sig.nslots, 1))()
        _lib.call("tf_signal_read", self.team.handle, int(pe), int(sig.base), int(sig.nslots), out)
        return np.frombuffer(bytes(out), dtype=np.uint64)[: sig.nslots].astype(np.int64)

    def symm_at(self, handle: SymmHandle, pe: int) -> RemoteRegion:
        self._check_pe(pe)
        return RemoteRegion(self, handle, pe)

    remote_ptr = symm_at

    # ------------------------------------------------------- signal plane ops
    def _slot(self, sig: SigHandle, idx: int, n: int, pe: int) -> int:
        self._check_pe(pe)
        if idx < 0 or idx + n > sig.nslots:
            raise ValueError(f"signal slots [{idx}, {idx + n}) exceed handle of {sig.nslots}")
        return sig.base + idx

    def ld(self, sig: SigHandle, idx: int, pe: int, scope: str = "gpu",
           semantic: str = "acquire") -> int:
        _check_scope_semantic(scope, semantic)
        self._slot(sig, idx, 1, pe)
        torch.cuda.synchronize(self.team.devices[pe])
        return int(self.sig_view(SigHandle(sig.base + idx, 1), pe)[0])

    def st(self, sig: SigHandle, idx: int, value: int, pe: int, scope: str = "gpu",
           semantic: str = "relaxed", name: str = "st", stream=None) -> None:
        _check_scope_semantic(scope, semantic)
        slot = self._slot(sig, idx, 1, pe)
        _lib.call("tf_signal_op", self.team.handle, int(pe), slot, int(value), 0, _stream_ptr(stream))

    def notify(self, sig: SigHandle, idx: int, pe: int, value: int, semantic: str = "release",
               stream=None) -> None:
        self.st(sig, idx, value, pe, scope="sys", semantic=semantic, name="notify", stream=stream)

    def atomic_add(self, sig: SigHandle, idx: int, val: int, pe: int, semantic: str = "release",
                   scope: str = "gpu", stream=None, fetch: bool = True):
        """Release add on a signal slot (shmem.py:184-194).  With fetch=True (the
        reference's contract) it returns the old value, which drains the stream;
        fetch=False is the stream-ordered form and returns None."""
        _check_scope_semantic(scope, semantic)
        slot = self._slot(sig, idx, 1, pe)
        if not fetch:
            _lib.call("tf_signal_op", self.team.handle, int(pe), slot, int(val), 1, _stream_ptr(stream))
            return None
        old = C.c_uint64()
        _lib.call("tf_signal_fetch_add", self.team.handle, int(pe), slot, int(val) & (2 ** 64 - 1),
                  C.byref(old), _stream_ptr(stream))
        return int(old.value)

    def atomic_cas(self, sig: SigHandle, idx: int, cmp: int, val: int, pe: int,
                   semantic: str = "release", scope: str = "gpu", stream=None) -> int:
        """Compare-and-swap of a signal slot (shmem.py:196-206); returns the old value.
        Synchronous (the caller needs the answer), executed on the device at .sys scope."""
        _check_scope_semantic(scope, semantic)
        slot = self._slot(sig, idx, 1, pe)
        old = C.c_uint64()
        _lib.call("tf_signal_cas", self.team.handle, int(pe), slot, int(cmp) & (2 ** 64 - 1),
                  int(val) & (2 ** 64 - 1), C.byref(old), _stream_ptr(stream))
        return int(old.value)

    def wait(self, sig: SigHandle, idx: int, num_slots: int, pe: int, scope: str = "gpu",
             semantic: str = "acquire", value: int = 1, note=None, stream=None,
             cmp: str = "eq") -> Token:
        """Stream waits until every slot in [idx, idx+num_slots) == value (the
        reference's semantics, shmem.py:208-235); cmp="ge" waits for >= value
        (epoch-valued flags that only grow)."""
        _check_scope_semantic(scope, semantic)
        if num_slots < 1:
            raise ValueError("wait needs num_slots >= 1")
        if cmp not in ("eq", "ge"):
            raise ValueError(f"cmp must be 'eq' or 'ge', got {cmp!r}")
        slot = self._slot(sig, idx, num_slots, pe)
        _lib.call("tf_signal_wait_cmp", self.team.handle, int(pe), slot, int(num_slots), int(value),
                  1 if cmp == "eq" else 0, _stream_ptr(stream))
        return Token(pe=int(pe), slot=slot, num_slots=int(num_slots))

    def reset_signals(self, sig: SigHandle, pe: int, stream=None) -> None:
        slot = self._slot(sig, 0, sig.nslots, pe)
        _lib.call("tf_signal_reset", self.team.handle, int(pe), slot, int(sig.nslots), _stream_ptr(stream))

    # ---------------------------------------------------------- data plane ops
    def putmem(self, dest: RemoteRegion, dest_off: int, src: torch.Tensor, *, from_pe: int = 0,
               note: str = "putmem", stream=None):
        nbytes = src.numel() * src.element_size()
        _check_range(dest.handle, dest_off, nbytes)
        src = src.contiguous()
        _lib.call("tf_putmem", self.team.handle, int(dest.pe), dest.handle.offset + int(dest_off),
                  src.data_ptr(), nbytes, _stream_ptr(stream))

    def getmem(self, dst: torch.Tensor, src: RemoteRegion, src_off: int, *, from_pe: int = 0,
               note: str = "getmem", stream=None):
        if not dst.is_contiguous():
            raise ValueError("getmem destination must be contiguous")
        nbytes = dst.numel() * dst.element_size()
        _check_range(src.handle, src_off, nbytes)
        _lib.call("tf_getmem", self.team.handle, int(src.pe), src.handle.offset + int(src_off),
                  dst.data_ptr(), nbytes, _stream_ptr(stream))

    def putmem_signal(self, dest: RemoteRegion, dest_off: int, src: torch.Tensor, sig: SigHandle,
                      idx: int, value: int, sig_op: str = "set", *, from_pe: int = 0,
                      note: str = "putmem_signal", stream=None):
        if sig_op not in ("set", "add"):
            raise ValueError(f"sig_op must be 'set' or 'add', got {sig_op!r}")
        slot = self._slot(sig, idx, 1, dest.pe)
        nbytes = src.numel() * src.element_size()
        _check_range(dest.handle, dest_off, nbytes)
        src = src.contiguous()
        _lib.call("tf_putmem_signal", self.team.handle, int(dest.pe),
                  dest.handle.offset + int(dest_off), src.data_ptr(), nbytes, slot, int(value),
                  1 if sig_op == "add" else 0, _stream_ptr(stream))

    putmem_nbi = putmem
    getmem_nbi = getmem

    def putmem_strided(self, dest: RemoteRegion, dest_off: int, src2d: torch.Tensor, dest_pitch: int, *,
                       from_pe: int = 0, note: str = "putmem", stream=None):
        """2-D block into rows `dest_pitch` bytes apart (shmem.py:253-268), one 2-D copy."""
        if src2d.dim() != 2:
            raise ValueError("putmem_strided needs a 2-D source block")
        rows = src2d.shape[0]
        row_nbytes = src2d.shape[1] * src2d.element_size()
        if rows:
            _check_range(dest.handle, dest_off, (rows - 1) * dest_pitch + row_nbytes)
        if rows == 0 or row_nbytes == 0:
            return
        if dest_pitch < row_nbytes:
            raise ValueError("dest_pitch smaller than a row")
        src_pitch = src2d.stride(0) * src2d.element_size()
        if src2d.stride(1) != 1:
            src2d = src2d.contiguous()
            src_pitch = row_nbytes
        _lib.call("tf_putmem_strided", self.team.handle, int(dest.pe), dest.handle.offset + int(dest_off),
                  int(dest_pitch), src2d.data_ptr(), int(src_pitch), int(row_nbytes), int(rows),
                  _stream_ptr(stream))

    def fence(self, from_pe: int) -> None:
        """Ordering of puts from one stream is already issue-order (copy engine queue)."""
        self._check_pe(from_pe)

    # ------------------------------------------------------------------ node-team collectives
    # multimem_ld_reduce / multimem_st (shmem.py:335-385): on one NVSwitch box the node
    # team is every PE.  The reduce reads each PE's copy over P2P and sums in ascending
    # rank order (bf16 in fp32, fp32, int64 exact); the broadcast is one copy-engine
    # transfer per PE.  Host-initiated and stream-ordered; results are device tensors.
    _RED_CODES = {torch.bfloat16: 0, torch.float32: 1, torch.int64: 2}

    def _pe_device(self, pe: int) -> int:
        return self.team.devices[pe] if self.team.rank is None else self.team.devices[self.team.rank]

    def multimem_ld_reduce(self, handle: SymmHandle, offset: int, dtype, count: int, pe: int,
                           stream=None) -> torch.Tensor:
        self._check_pe(pe)
        tdt = _torch_dtype(dtype)
        if tdt not in self._RED_CODES:
            raise ValueError(f"multimem_ld_reduce supports bf16, fp32, int64; got {tdt}")
        isz = torch.empty(0, dtype=tdt).element_size()
        _check_range(handle, offset, count * isz)
        dev = self._pe_device(pe)
        out = torch.empty(int(count), dtype=tdt, device=f"cuda:{dev}")
        fn = "tf_nvls_reduce" if handle.space == "nvls" else "tf_team_reduce"
        with torch.cuda.device(dev):
            _lib.call(fn, self.team.handle, int(pe), handle.offset + int(offset),
                      self._RED_CODES[tdt], int(count), out.data_ptr(), _stream_ptr(stream))
        return out

    def multimem_st(self, handle: SymmHandle, offset: int, vec, pe: int, stream=None) -> None:
        self._check_pe(pe)
        dev = self._pe_device(pe)
        v = vec if isinstance(vec, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(vec))
        v = v.contiguous().to(f"cuda:{dev}")
        nbytes = v.numel() * v.element_size()
        _check_range(handle, offset, nbytes)
        fn = "tf_nvls_broadcast" if handle.space == "nvls" else "tf_team_broadcast"
        with torch.cuda.device(dev):
            _lib.call(fn, self.team.handle, int(pe), handle.offset + int(offset),
                      v.data_ptr(), nbytes, _stream_ptr(stream))
        if stream is None:
            torch.cuda.synchronize(dev)  # v may be a temporary

    def multimem_ld_reduce_block(self, handle: SymmHandle, pe: int, dtype, shape, row0: int, nrows: int,
                                 col0: int, ncols: int, stream=None) -> torch.Tensor:
        """Team sum of rows [row0, row0 + nrows) x cols [col0, col0 + ncols) of a
        matrix laid out with `shape` in the region (shmem.py:363-375)."""
        rows, cols = shape
        if row0 < 0 or nrows < 0 or row0 + nrows > rows or col0 < 0 or ncols < 0 or col0 + ncols > cols:
            raise ValueError(f"block [{row0}:{row0 + nrows}, {col0}:{col0 + ncols}] outside {tuple(shape)}")
        isz = torch.empty(0, dtype=_torch_dtype(dtype)).element_size()
        full = self.multimem_ld_reduce(handle, row0 * cols * isz, dtype, nrows * cols, pe, stream)
        return full.view(nrows, cols)[:, col0:col0 + ncols].clone()

    def multimem_st_block(self, handle: SymmHandle, pe: int, block, shape, row0: int, col0: int) -> None:
        """Write a 2-D block into every PE's copy (shmem.py:377-385)."""
        self._check_pe(pe)
        b = block if isinstance(block, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(block))
        r1, c1 = row0 + b.shape[0], col0 + b.shape[1]
        if row0 < 0 or col0 < 0 or r1 > shape[0] or c1 > shape[1]:
            raise ValueError(f"block [{row0}:{r1}, {col0}:{c1}] outside {tuple(shape)}")
        for r in range(self.topology.world_size):
            dst = self.view(handle, r, b.dtype, shape)
            dst[row0:r1, col0:c1].copy_(b.to(dst.device))

    def node_barrier(self, rank: int | None = None, barrier=None, stream=None):
        """Rendezvous of the node team (shmem.py:329-331): every PE on one box."""
        return self.barrier_all(rank, stream)

    def barrier_all(self, rank: int | None = None, stream=None):
        """All-rank rendezvous ordered after every prior op on the rank's stream.
        With rank=None every local PE arrives and then waits (single-process team)."""
        ranks = self.team.local_ranks() if rank is None else [rank]
        for r in ranks:
            self._check_pe(r)
            with torch.cuda.device(self.team.devices[r]):
                _lib.call("tf_barrier_arrive", self.team.handle, r, _stream_ptr(stream))
        for r in ranks:
            with torch.cuda.device(self.team.devices[r]):
                _lib.call("tf_barrier_wait", self.team.handle, r, _stream_ptr(stream))

    # sync_all (shmem.py:324-327) is rendezvous-only in the reference; here every put
    # is stream-ordered before the arrival, so the rendezvous also drains them.
    sync_all = barrier_all


def _check_scope_semantic(scope: str, semantic: str):
    if scope not in SCOPES:
        raise ValueError(f"invalid scope {scope!r}; expected one of {SCOPES}")
    if semantic not in SEMANTICS:
        raise ValueError(f"invalid semantic {semantic!r}; expected one of {SEMANTICS}")


def _check_range(handle: SymmHandle, off: int, nbytes: int):
    if off < 0 or off + nbytes > handle.nbytes:
        raise ValueError(f"range [{off}, {off + nbytes}) exceeds region of {handle.nbytes} bytes")


_NP2T = {
    np.dtype(np.uint8): torch.uint8, np.dtype(np.int8): torch.int8,
    np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64,
    np.dtype(np.float32): torch.float32, np.dtype(np.float16): torch.float16,
    np.dtype(np.float64): torch.float64, np.dtype(np.uint64): torch.uint64,
}


def _torch_dtype(dtype) -> torch.dtype:
    if isinstance(dtype, torch.dtype):
        return dtype
    return _NP2T[np.dtype(dtype)]
