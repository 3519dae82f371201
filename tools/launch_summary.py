"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by
kernel and grid: launches, total device time, share.  Markdown to stdout.

    python tools/launch_summary.py gpurun_out/r03_launches.csv [--last N]
"""
import csv
import sys
from collections import OrderedDict

path = sys.argv[1]
last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else None
rows = []
with open(path) as fh:
    lines = [l for l in fh if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    ns = float(r["Metric Value"].replace(",", ""))
    us = ns / 1e3 if r["Metric Unit"] == "ns" else ns * (1e3 if r["Metric Unit"] == "msecond" else 1)
    rows.append((r["Kernel Name"], r["Grid Size"], us))
if last:
    rows = rows[-last:]
agg = OrderedDict()
for name, grid, us in rows:
    short = name.split("(")[0].replace("void ", "")
    k = f"`{short}` grid {grid}"
    c, t = agg.get(k, (0, 0.0))
    agg[k] = (c + 1, t + us)
tot = sum(t for _, t in agg.values())
print("| kernel | launches | total us | share |")
print("|---|---|---|---|")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| {k} | {c} | {t:.1f} | {100 * t / tot:.1f}% |")
print(f"\nTotal: {tot:.1f} us over {len(rows)} launches.")
