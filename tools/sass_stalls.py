"""Stall-reason totals per kernel from a gzipped `ncu --page source --csv --print-source sass` dump
(usage: sass_stalls.py dump.csv.gz kernel-substring)."""
import collections
import csv
import gzip
import sys

rows = list(csv.reader(gzip.open(sys.argv[1], "rt")))
ks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]
        ks.append(cur)
    elif r and r[0] == "Address":
        cur[1] = r
    elif cur and cur[1] and len(r) > 5:
        cur[2].append(r)
for name, h, body in ks:
    if sys.argv[2] not in name:
        continue
    sc = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
    tot = collections.Counter()
    for r in body:
        for i in sc:
            if r[i].isdigit():
                tot[h[i]] += int(r[i])
    s = sum(tot.values())
    print(name[:90], s)
    print("  " + ", ".join(f"{k[6:]} {v / s * 100:.1f}%" for k, v in tot.most_common(10)))
