"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) into
profiles/: per-launch lines in order plus per-kernel totals and shares.
    python tools/launch_summary.py gpurun_out/launches.csv "<command>" > profiles/r01_launches.txt"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, out = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        u = r[hdr.index("Metric Unit")]
        v = float(r[hdr.index("Metric Value")].replace(",", ""))
        us = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}[u]
        out.append((r[hdr.index("Kernel Name")], us))
total = sum(t for _, t in out)
ours = sum(t for k, t in out if "tf::" in k)
print(f"# {sys.argv[2] if len(sys.argv) > 2 else ''}")
print("# cold-cache serialised per-launch times: compare SHARES, not absolutes")
print(f"# {len(out)} launches, total {total:.1f} us; tilefuse kernels {ours:.1f} us ({100 * ours / total:.1f}%)")
agg = collections.defaultdict(lambda: [0, 0.0])
for k, t in out:
    agg[k[:110]][0] += 1
    agg[k[:110]][1] += t
print("# per kernel: launches, total us, share")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"#  {n:4d} {t:11.1f} us {100 * t / total:5.1f}%  {k}")
for k, t in out:
    print(f"{t:12.1f} us {100 * t / total:5.1f}%  {k[:140]}")
