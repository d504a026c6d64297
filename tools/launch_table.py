"""Per-kernel table (count, mean us, share, DRAM MB per launch, FP64 pipe %) of an
ncu launch-list CSV (usage: launch_table.py launches.csv [steps])."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
L = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    L.setdefault(r[idi], {"name": r[ki]})
    try:
        L[r[idi]][r[mi]] = float(r[vi].replace(",", ""))
    except ValueError:
        pass
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for l in L.values():
    n = l["name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
    a = agg[n]
    a[0] += 1
    a[1] += l.get("gpu__time_duration.sum", 0.0)
    a[2] += l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)
    a[3] += l.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0.0)
tot = sum(a[1] for a in agg.values())
steps = int(sys.argv[2]) if len(sys.argv) > 2 else None
print("| kernel | launches | us / launch | share | DRAM MB / launch | FP64 pipe % |")
print("|---|---|---|---|---|---|")
for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| {n} | {a[0]} | {a[1] / a[0] / 1e3:.1f} | {a[1] / tot * 100:.1f} % | {a[2] / a[0] / 1e6:.1f} | {a[3] / a[0]:.1f} |")
if steps:
    print(f"\nper step: {tot / steps / 1e3:.1f} us, DRAM {sum(a[2] for a in agg.values()) / steps / 1e6:.1f} MB")
