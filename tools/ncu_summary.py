"""Summarise an `ncu --page raw --csv` export into a markdown table.

usage: python tools/ncu_summary.py raw.csv [more.csv ...] > summary.md
"""
import csv
import sys

METRICS = [
    ("time_us", "gpu__time_duration.sum", 1.0),
    ("dram_rd_MB", "dram__bytes_read.sum", None),
    ("dram_wr_MB", "dram__bytes_write.sum", None),
    ("dram_%peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed|dram__throughput.avg.pct_of_peak_sustained_elapsed|FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("sm_%peak", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("warps_act_%", "sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    ("regs", "launch__registers_per_thread", 1.0),
    ("fp64_pipe_%", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    ("smem_wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1.0),
    ("grid", "launch__grid_size", 1.0),
]


def to_mb(val, unit):
    v = float(val.replace(",", ""))
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "KB": 1e-3, "MB": 1.0, "GB": 1e3, "B": 1e-6}
    return v * scale.get(unit.strip(), 1.0)


def main(paths):
    print("| kernel | " + " | ".join(m[0] for m in METRICS) + " |")
    print("|---" * (len(METRICS) + 1) + "|")
    for p in paths:
        with open(p) as f:
            rows = list(csv.reader(f))
        hdr, units = rows[0], rows[1]
        idx = {h: i for i, h in enumerate(hdr)}
        for r in rows[2:]:
            name = r[idx["Kernel Name"]]
            name = name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
            cells = []
            for label, keys, _ in METRICS:
                key = next((k for k in keys.split("|") if k in idx), None)
                if key is None:
                    cells.append("-")
                    continue
                val = r[idx[key]]
                if label.endswith("_MB"):
                    cells.append(f"{to_mb(val, units[idx[key]]):.1f}")
                elif label == "time_us":
                    u = units[idx[key]].strip()
                    v = float(val.replace(",", ""))
                    v = v / 1e3 if u == "nsecond" else v * 1e3 if u == "msecond" else v
                    cells.append(f"{v:.1f}")
                else:
                    cells.append(val)
            print(f"| `{name}` | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1:])
