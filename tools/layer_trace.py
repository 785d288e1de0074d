"""Per-layer timeline of the config-5 megakernel from its device trace
(python tools/layer_trace.py [tokens]); prints, per layer, the span and the
mean task time split into dependency wait and work."""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2605_02953_b200 import build_topology
from paper_2605_02953_b200 import layer as L

T = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
H, HQ, HKV, FF = 8192, 64, 8, 28672
prog = L.llama_layer_program(build_topology(1, 1), T, H, HQ, HKV, FF, seq_len=T)
r = L.LayerRunner(prog, device=0)
g = torch.Generator().manual_seed(1)
for t in prog.tensors:
    v = r.view(t.name)
    v.copy_((torch.randn(v.shape, generator=g) * (0.02 if t.name.startswith("w") else 1)).to(v.dtype))
for _ in range(2):
    r.run()
torch.cuda.synchronize()
r.enable_trace()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
r.run()
e1.record()
torch.cuda.synchronize()
r.check()
ms = e0.elapsed_time(e1)
tr = np.array(r.trace(), dtype=np.int64)
t0 = tr[:, 3].min()
names = [f"{lid}:{op}" for lid, op in r.built.layer_ops.items()]
rep = {"ms_total": ms, "layers": []}
for lid, nm in enumerate(names):
    sel = tr[tr[:, 1] == lid]
    rep["layers"].append({
        "layer": nm, "tasks": int(len(sel)),
        "start_us": round((sel[:, 3].min() - t0) / 1e3, 1), "end_us": round((sel[:, 5].max() - t0) / 1e3, 1),
        "mean_wait_us": round(float(np.mean(sel[:, 4] - sel[:, 3])) / 1e3, 2),
        "mean_task_us": round(float(np.mean(sel[:, 5] - sel[:, 4])) / 1e3, 2),
        "sum_task_ms_over_ctas": round(float(np.sum(sel[:, 5] - sel[:, 4])) / 1e6 / r.num_sms, 3)})
# wave coherence of each layer: the k-th task of a layer in every CTA's queue belongs to
# wave k of the round-robin queues; spread of their start (deps satisfied) times
for lid, nm in enumerate(names):
    sel = tr[tr[:, 1] == lid]
    if not len(sel) or "linear" not in nm:
        continue
    waves = {}
    for c in np.unique(sel[:, 0]):
        rows = sel[sel[:, 0] == c]
        rows = rows[np.argsort(rows[:, 3])]
        for k, row in enumerate(rows):
            waves.setdefault(k, []).append(row[4])
    task = float(np.mean(sel[:, 5] - sel[:, 4]))
    spreads = [(max(v) - min(v)) / task for k, v in sorted(waves.items()) if len(v) > 1]
    rep.setdefault("wave_start_spread_tasks", {})[nm] = {
        "median": round(float(np.median(spreads)), 2), "max": round(float(np.max(spreads)), 2),
        "waves": len(spreads)}
busy_end = np.array([tr[tr[:, 0] == c][:, 5].max() - t0 for c in range(r.num_sms)]) / 1e3
rep["cta_finish_us"] = {"min": float(busy_end.min()), "median": float(np.median(busy_end)),
                        "max": float(busy_end.max())}
print(json.dumps(rep, indent=1))
