"""Per-key-tile timeline of one attention CTA (SM clock stamps).  Needs a build
with -DTF_ATTN_TRACE:  TF_NVCC_EXTRA=-DTF_ATTN_TRACE python tools/attn_trace.py"""

import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as g  # noqa: E402

g.build()
import bench  # noqa: E402
from paper_2605_02953_b200 import _lib  # noqa: E402

print(bench.bench_attention(0, 2, {}))
buf = np.zeros((512, 20), dtype=np.int64)
lib = _lib.lib() if callable(getattr(_lib, "lib", None)) else _lib._LIB
assert lib.tf_attn_trace_dump(buf.ctypes.data_as(C.POINTER(C.c_longlong))) == 0
t0 = buf[0, 0]
names = ["gotS_A", "gotS_B", "relP_A", "relP_B", "PV_A", "PV_B", "S+_A", "S+_B", "mmaKV", "ldK", "ldV", "mmaV", "relP_A1", "relP_B1", "relP_A0", "relP_B0", "preHalfA", "postHalfA", "-", "-"]
print("j  " + " ".join(f"{n:>8s}" for n in names) + "   period")
for j in list(range(0, 6)) + list(range(100, 112)) + list(range(250, 256)):
    row = buf[j] - buf[j, 0]
    per = buf[j + 1, 0] - buf[j, 0] if j + 1 < 256 else 0
    print(f"{j:3d} " + " ".join(f"{v:8d}" for v in row) + f"   {per:6d}")
mid = buf[20:240]
per = np.diff(buf[20:241, 0])
print("median period", np.median(per))
for i, n in enumerate(names):
    print(f"median {n:8s} - gotS_A: {np.median(mid[:, i] - mid[:, 0]):8.0f}")
