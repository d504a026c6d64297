#!/usr/bin/env bash
# Session-4: fused eigenvector stage of the QL tier (SDP_TRD_FUSEVEC) -- parity, A/B bench, launch list.
set -u
OUT=gpurun_out/s4b
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/rc.txt"
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -k "trd or batch or psd" > "$OUT/pytest_trd.log" 2>&1; echo "pytest rc=$?" >> "$OUT/rc.txt"
for fv in 1 0 1 0; do
  SDP_TRD_FUSEVEC=$fv timeout 600 python bench.py --workload cfg4 --steps 20 --no-cpu > "$OUT/bench_cfg4_fv$fv.json" 2> "$OUT/bench_cfg4_fv$fv.err"
  python -c "import json;d=json.loads(open('$OUT/bench_cfg4_fv$fv.json').read().strip().splitlines()[-1]);print('fv=$fv',d['value'],d['ms_per_step'])" >> "$OUT/ab.txt" 2>&1
done
timeout 900 python bench.py --workload cfg3 --steps 100 --warmup 10 --no-cpu > "$OUT/bench_cfg3.json" 2> "$OUT/bench_cfg3.err"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
    --log-file "$OUT/launches_cfg4.csv" python bench.py --workload cfg4 --steps 2 --warmup 3 --no-cpu > "$OUT/ncu_l4.log" 2>&1
echo done >> "$OUT/rc.txt"
