"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per
kernel name, launches and total / mean / max duration, in launch order of first
appearance. usage: python tools/launch_summary.py launches.csv [> summary.md]"""
import csv
import sys
from collections import OrderedDict

rows = []
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") == "gpu__time_duration.sum":
        rows.append((r["Kernel Name"], r["Grid Size"], r["Block Size"], float(r["Metric Value"].replace(",", ""))))
agg = OrderedDict()
for name, grid, block, ns in rows:
    short = name.split("(")[0].replace("void ", "")
    key = (short, grid, block)
    a = agg.setdefault(key, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += ns
    a[2] = max(a[2], ns)
tot = sum(v[1] for v in agg.values())
print(f"# launch list: {len(rows)} launches, {tot / 1e6:.3f} ms of kernel time\n")
print("| kernel | grid | block | launches | total ms | mean us | max us | share |")
print("|---|---|---|---|---|---|---|---|")
for (short, grid, block), (n, s, mx) in agg.items():
    print(f"| `{short}` | {grid} | {block} | {n} | {s / 1e6:.3f} | {s / n / 1e3:.1f} | {mx / 1e3:.1f} | {s / tot:.1%} |")
