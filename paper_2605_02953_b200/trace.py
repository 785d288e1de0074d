"""Device-event traces in the reference's schema.

The reference records simulated TraceEvents (ovs/simengine.py:56-73) and
exports them as Chrome 'X' events (:372-389).  Here the GEMM kernels write
per-tile events stamped with %globaltimer into a device ring
(`tf_trace_enable`), which `collect()` converts to the same TraceEvent /
Trace structure so the reference's protocol assertions (a straddling tile
waits on both chunks, gather order starts at the local chunk) can be checked
against the real kernels, and `export_chrome_trace` writes the same JSON.

Kinds: "wait" (name wait_chunks: slot = first chunk, num_slots), "compute"
(name gemm_tile: MMA issue window of a tile), "store" (name epilogue), "signal"
(name atomic_add: a GEMM-RS producer bumped owner `pe`'s row-block counter `slot`
to `value`; name segment_ready: owner `pe` saw counter `slot` complete).
Times are seconds relative to the first event.
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field

import numpy as np

from . import _lib

_KINDS = {1: ("wait", "wait_chunks"), 2: ("compute", "gemm_tile"), 3: ("store", "epilogue"),
          4: ("signal", "atomic_add"), 5: ("signal", "segment_ready")}


@dataclass(frozen=True)
class TraceEvent:
    rank: int
    worker: str
    worker_id: int
    kind: str
    t_start: float
    t_end: float
    payload: dict


@dataclass
class Trace:
    events: list = field(default_factory=list)
    seed: int = 0

    def by_kind(self, kind: str) -> list:
        return [e for e in self.events if e.kind == kind]


def enable(device: int = 0, capacity: int = 1 << 20) -> None:
    _lib.call("tf_trace_enable", int(device), int(capacity))


def disable(device: int = 0) -> None:
    _lib.call("tf_trace_disable", int(device))


def collect(device: int = 0, capacity: int = 1 << 20) -> Trace:
    """Read (and clear) the device ring; synchronise the device first."""
    buf = np.zeros((capacity, 4), dtype=np.uint64)
    n = C.c_int64()
    _lib.call("tf_trace_read", int(device), buf.ctypes.data, int(capacity), C.byref(n))
    rec = buf[: n.value]
    if not len(rec):
        return Trace([])
    t0 = int(rec[:, 1].min())
    events = []
    for w0, ts, te, pl in rec.tolist():
        kind, name = _KINDS.get(int(w0) >> 56, ("unknown", "unknown"))
        rank = (int(w0) >> 48) & 0xFF
        cta = (int(w0) >> 32) & 0xFFFF
        tile = int(w0) & 0xFFFFFFFF
        if kind == "wait":
            payload = {"name": name, "tile": tile, "slot": int(pl) >> 32, "num_slots": int(pl) & 0xFFFFFFFF}
        elif kind == "signal":
            # RS row-block counter: bump by producer `rank` (value = count after it), or the
            # owner observing it complete (gemm_rs.py:155-161 atomic_add / segment_ready)
            payload = {"name": name, "slot": tile, "pe": int(pl) >> 32, "value": int(pl) & 0xFFFFFFFF}
        else:
            payload = {"name": name, "tile": tile, "pid_m": int(pl) >> 32, "pid_n": int(pl) & 0xFFFFFFFF}
        events.append(TraceEvent(rank, f"cta{cta}", cta, kind, (int(ts) - t0) * 1e-9,
                                 (int(te) - t0) * 1e-9, payload))
    events.sort(key=lambda e: (e.t_start, e.rank, e.worker_id))
    return Trace(events)


def export_chrome_trace(trace: Trace, path) -> None:
    """Chrome 'X' duration events, ts/dur in us, pid=rank, tid=worker id -- the
    reference's schema (simengine.py:372-389)."""
    out = []
    for e in trace.events:
        out.append({"name": str(e.payload.get("name", e.kind)), "cat": e.kind, "ph": "X",
                    "ts": e.t_start * 1e6, "dur": (e.t_end - e.t_start) * 1e6,
                    "pid": e.rank, "tid": e.worker_id,
                    "args": {k: v for k, v in sorted(e.payload.items()) if k != "name"}})
    with open(path, "w", encoding="utf-8") as f:
        f.write(json.dumps(out, separators=(",", ":"), sort_keys=True))
