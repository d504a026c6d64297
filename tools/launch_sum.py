"""Per-kernel totals of an ncu --csv launch list (gpu__time_duration.sum)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
d = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        d[r[ki][:60]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{k:60s} n={len(v):4d} mean={sum(v) / len(v) / 1e3:9.1f}us share={sum(v) / tot:.3f}")
