"""Print metric name / unit / value rows of ncu --csv --log-file outputs.
    python tools/ncu_csv_metrics.py file.csv [...]"""
import csv
import sys

for path in sys.argv[1:]:
    print(f"== {path}")
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for row in csv.DictReader(lines):
        name = row.get("Kernel Name", "")[:60]
        print(f"  {row.get('Metric Name',''):70s} {row.get('Metric Unit',''):10s} {row.get('Metric Value','')}   [{name}]")
