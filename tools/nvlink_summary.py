"""Per-kernel NVLink / DRAM totals from tools/nvlink_capture.sh's per-process ncu CSVs."""
import collections
import csv
import glob
import io
import os
import sys


def main():
    d = sys.argv[1]
    for path in sorted(glob.glob(os.path.join(d, "launches_*.csv"))):
        text = open(path, encoding="utf-8", errors="replace").read()
        start = text.find('"ID"')
        if start < 0:
            print(f"{path}: no launches")
            continue
        rows = list(csv.DictReader(io.StringIO(text[start:])))
        acc = collections.defaultdict(lambda: collections.defaultdict(float))
        cnt = collections.Counter()
        for r in rows:
            name = r["Kernel Name"].split("(")[0][:70]
            key = (name, r["Metric Name"])
            try:
                v = float(r["Metric Value"].replace(",", ""))
            except ValueError:
                continue
            unit = r.get("Metric Unit", "")
            scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e3, "msecond": 1e6}.get(unit, 1.0)
            acc[name][r["Metric Name"]] += v * scale
            if r["Metric Name"] == "gpu__time_duration.sum":
                cnt[name] += 1
        print(f"== {os.path.basename(path)}")
        for name, m in sorted(acc.items(), key=lambda kv: -kv[1].get("gpu__time_duration.sum", 0)):
            t_ns = m.get("gpu__time_duration.sum", 0.0)
            tx = m.get("nvltx__bytes_data_user.sum", 0.0)
            rx = m.get("nvlrx__bytes_data_user.sum", 0.0)
            gbps = (tx / t_ns) if t_ns else 0.0  # bytes/ns = GB/s
            print(f"{cnt[name]:4d}x {name:70s} {t_ns / 1e3:10.1f} us  nvl tx {tx / 1e6:9.1f} MB"
                  f"  rx {rx / 1e6:9.1f} MB  tx {gbps:7.1f} GB/s  dram r {m.get('dram__bytes_read.sum', 0) / 1e6:9.1f} MB")


if __name__ == "__main__":
    main()
