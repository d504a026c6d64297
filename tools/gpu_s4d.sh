#!/usr/bin/env bash
# Session-4: QL-tier eigenvector kernel with the cluster CTAs first (SDP_TRD_INVIT_ORDER) -- parity, A/B bench, launch list.
set -u
OUT=gpurun_out/s4d
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/rc.txt"
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -k "trd or batch or psd" > "$OUT/pytest_trd.log" 2>&1; echo "pytest rc=$?" >> "$OUT/rc.txt"
for o in 1 0 1 0; do
  SDP_TRD_INVIT_ORDER=$o timeout 600 python bench.py --workload cfg4 --steps 20 --no-cpu > "$OUT/bench_cfg4_o$o.json" 2> "$OUT/bench_cfg4_o$o.err"
  python -c "import json;d=json.loads(open('$OUT/bench_cfg4_o$o.json').read().strip().splitlines()[-1]);print('order=$o',d['value'],d['ms_per_step'])" >> "$OUT/ab.txt" 2>&1
done
SDP_TRD_INVIT_ORDER=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
    --log-file "$OUT/launches_cfg4.csv" python bench.py --workload cfg4 --steps 2 --warmup 3 --no-cpu > "$OUT/ncu_l4.log" 2>&1
echo done >> "$OUT/rc.txt"
