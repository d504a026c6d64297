"""Per-kernel summary of an `ncu --metrics ... --csv --log-file` launch list.
usage: python tools/launch_summary.py launches.csv [skip_setup_kernels=1]"""
import collections
import csv
import sys

SETUP = ("k_gj_sweep", "k_gj_diag", "k_syrk_dmma", "k_syrk_dense", "k_place_dense", "k_transpose", "k_mask_cols")


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ix = {k: j for j, k in enumerate(h)}
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for r in rows[hdr + 1:]:
        if len(r) < len(h):
            continue
        n = r[ix["Kernel Name"]].split("(")[0].replace("void ", "").replace("unnamed>::", "").replace("sdp::", "")
        n = n.lstrip("<")
        if n.startswith("at::"):
            n = "[torch] " + n.split("<")[0] + " (bench L2 flush)"
        m = r[ix["Metric Name"]]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        agg[n][m] += v
        if m == "gpu__time_duration.sum":
            cnt[n] += 1
    tot = sum(a["gpu__time_duration.sum"] for n, a in agg.items() if not n.startswith(SETUP + ("[torch]",)))
    print(f"| kernel | launches | us / launch | share of non-setup time | DRAM MB / launch | FP64 pipe % |")
    print("|---|---|---|---|---|---|")
    for n, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
        c = cnt[n]
        t = a["gpu__time_duration.sum"] / c / 1000
        share = ("setup" if n.startswith(SETUP) else "bench" if n.startswith("[torch]")
                 else f"{100 * a['gpu__time_duration.sum'] / tot:.1f} %")
        dram = (a.get("dram__bytes_read.sum", 0) + a.get("dram__bytes_write.sum", 0)) / c / 1e6
        fp = a.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
        fp = f"{fp / c:.1f}" if fp is not None else "-"
        print(f"| {n} | {c} | {t:.1f} | {share} | {dram:.1f} | {fp} |")


if __name__ == "__main__":
    main(sys.argv[1])
