"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel and grid size.

usage: summarize_launches.py launches.csv [grid-filter]
Launches of different sizes (the bench's batched step vs the e2e path's 16-curve chunks) are
kept apart; shares are computed over the largest-grid launch set of each kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hdr_i]
data = rows[hdr_i + 1:]
ki, vi, ui, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit"), hdr.index("Grid Size")
agg = collections.defaultdict(list)
for r in data:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")[:40]
    agg[(name, r[gi])].append(float(r[vi].replace(",", "")))
print("unit", data[0][ui])
micro = ("k_imad", "k_imad_wide", "k_mmul2", "k_twiddles")
for (k, g), v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    if k in micro:
        continue
    print(f"{k:40s} grid={g:>18s} n={len(v):3d} mean={sum(v) / len(v):11.1f} min={min(v):11.1f}")
