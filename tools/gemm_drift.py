"""How far do the persistent GEMM clusters drift apart?  One traced launch (after
warm-up launches back to back) of the config-2 AG-shape GEMM: per cluster, its j-th
tile belongs to wave j; print per wave the spread of MMA start times across
clusters, in units of the mean tile time, and how many waves are in flight at once.
    python tools/gemm_drift.py [M N K]"""
import os
import statistics
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_02953_b200 import kernels as K  # noqa: E402
from paper_2605_02953_b200 import trace as T  # noqa: E402

m, n, k = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 28672, 8192)))
x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
w = (torch.randn(n, k, device="cuda") * k ** -0.5).to(torch.bfloat16)
out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
for _ in range(10):
    K.gemm(x, w, out, block_m=512, group_m=8)
T.enable(0)
K.gemm(x, w, out, block_m=512, group_m=8)
torch.cuda.synchronize()
tr = T.collect(0)
T.disable(0)
ev = tr.by_kind("compute")
per_cta = defaultdict(list)
for e in ev:
    per_cta[e.worker_id].append(e)
starts = defaultdict(list)
durs = []
for cta, es in per_cta.items():
    es.sort(key=lambda e: e.t_start)
    for j, e in enumerate(es):
        starts[j].append(e.t_start)
        durs.append(e.t_end - e.t_start)
tile = statistics.mean(durs)
print(f"{len(ev)} compute events from {len(per_cta)} CTAs; mean tile MMA window {tile * 1e6:.1f} us")
for j in sorted(starts):
    s = starts[j]
    print(f"wave {j:3d}: {len(s):3d} tiles, start spread {(max(s) - min(s)) / tile:5.2f} tiles, "
          f"first {min(s) * 1e6:8.1f} us")
end = max(e.t_end for e in ev)
print(f"kernel span {end * 1e6:.1f} us")

# per-CTA tile transitions: gap between consecutive MMA windows, and how long after a
# tile's MMA window its epilogue finished (drain tail)
comp = defaultdict(list)
epi = defaultdict(list)
for e in tr.events:
    if e.kind == "compute":
        comp[e.worker_id].append(e)
    elif e.kind == "store":
        epi[e.worker_id].append(e)
gaps, tails, edur = [], [], []
for cta, es in comp.items():
    es.sort(key=lambda e: e.t_start)
    for a, b in zip(es, es[1:]):
        gaps.append(b.t_start - a.t_end)
    ep = sorted(epi.get(cta, []), key=lambda e: e.t_start)
    for c, s in zip(es, ep):
        tails.append(s.t_end - c.t_end)
        edur.append(s.t_end - s.t_start)
if gaps:
    print(f"MMA gap between tiles: mean {statistics.mean(gaps) * 1e6:.2f} us, max {max(gaps) * 1e6:.2f} us")
if tails:
    print(f"epilogue end after MMA end: mean {statistics.mean(tails) * 1e6:.2f} us; epilogue event mean {statistics.mean(edur) * 1e6:.2f} us "
          f"({len(edur)} events from {len(epi)} CTAs)")
