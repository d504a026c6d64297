#!/usr/bin/env bash
# Session-4: QL-tier inverse iteration (clusters) with operands read eight rows ahead -- parity, bench, launch list.
set -u
OUT=gpurun_out/s4c
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/rc.txt"
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -k "trd or batch or psd" > "$OUT/pytest_trd.log" 2>&1; echo "pytest rc=$?" >> "$OUT/rc.txt"
for r in 1 2; do
  timeout 600 python bench.py --workload cfg4 --steps 20 --no-cpu > "$OUT/bench_cfg4_$r.json" 2> "$OUT/bench_cfg4_$r.err"
  python -c "import json;d=json.loads(open('$OUT/bench_cfg4_$r.json').read().strip().splitlines()[-1]);print('run $r',d['value'],d['ms_per_step'])" >> "$OUT/ab.txt" 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
    --log-file "$OUT/launches_cfg4.csv" python bench.py --workload cfg4 --steps 2 --warmup 3 --no-cpu > "$OUT/ncu_l4.log" 2>&1
echo done >> "$OUT/rc.txt"
