"""Per-key-tile timeline of the leader CTA of the S-double-buffered pair attention
kernel (SM clock stamps).  Needs -DTF_ATTN_TRACE:
    TF_NVCC_EXTRA=-DTF_ATTN_TRACE TF_ATTN_PAIR=2 python tools/attn_trace_pair2.py"""
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
assert _lib.lib().tf_attn_trace_dump(buf.ctypes.data_as(C.POINTER(C.c_longlong))) == 0
names = ["smx_gotS", "smx_relP", "mma_gotP", "mma_PV", "mma_S+2", "ld_K", "ld_V", "smx1_rel", "mma_top"]
print("j  " + " ".join(f"{n:>9s}" for n in names) + "   period(gotS)")
for j in list(range(0, 8)) + list(range(100, 112)) + list(range(250, 256)):
    row = buf[j, :9] - buf[j, 0]
    per = buf[j + 1, 0] - buf[j, 0] if j + 1 < 256 else 0
    print(f"{j:3d} " + " ".join(f"{v:9d}" for v in row) + f"   {per:6d}")
mid = buf[20:240, :9]
print("median period", np.median(np.diff(buf[20:241, 0])))
for i, nme in enumerate(names):
    print(f"median {nme:9s} - smx_gotS: {np.median(mid[:, i] - mid[:, 0]):8.0f}")
# cross-SM view (globaltimer ns): leader CTA slots 10.., peer CTA slots 15..
g0, g1 = buf[:, 10:15], buf[:, 15:20]
sel = slice(20, 240)
print("ns, median over j in [20,240):")
print("  leader gotS -> leader relP   ", np.median(g0[sel, 1] - g0[sel, 0]))
print("  peer   gotS -> peer relP     ", np.median(g1[sel, 1] - g1[sel, 0]))
print("  peer gotS - leader gotS      ", np.median(g1[sel, 0] - g0[sel, 0]))
print("  leader MMA gotP - leader relP", np.median(g0[sel, 2] - g0[sel, 1]))
print("  leader MMA gotP - peer relP  ", np.median(g0[sel, 2] - g1[sel, 1]))
print("  peer K load(j) - leader K load(j)", np.median(g1[sel, 3] - g0[sel, 3]))
print("  period (leader gotS)         ", np.median(np.diff(g0[20:241, 0])))
