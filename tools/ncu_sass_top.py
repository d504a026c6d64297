"""Top SASS instructions of one kernel in an ncu report by warp-stall samples
(usage: ncu_sass_top.py report.ncu-rep kernel-regex [n])."""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
si, ii, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
body = [r for r in rows[hi + 1:] if len(r) > ei and r[ii].isdigit()]
tot = sum(int(r[ii]) for r in body)
print(f"total samples {tot}, instructions {len(body)}")
idx = sorted(range(len(body)), key=lambda i: -int(body[i][ii]))[:n]
for i in sorted(idx):
    r = body[i]
    print(f"{i:5d} {int(r[ii]) / tot * 100:5.1f}% exec {r[ei]:>9s}  {r[si].strip()}")
