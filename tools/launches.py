"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list (per-kernel mean/count)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) > vi:
        agg[r[ki].split("(")[0][-48:]].append(float(r[vi].replace(",", "")))
for k, v in agg.items():
    print(f"{k:48s} n={len(v):3d} mean={sum(v) / len(v) / 1000:9.2f} us  min={min(v) / 1000:8.2f}")
