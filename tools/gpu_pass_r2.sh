#!/usr/bin/env bash
# Round-2 measurement pass: bench lines for every workload (+ the reference arm), ncu launch lists
# and full captures of the top kernels.  Output in gpurun_out/<tag>/.
set -u
TAG=${1:-r2pass}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/rc.txt"
timeout 900 python bench.py --paper-row > "$OUT/bench_cfg2.json" 2> "$OUT/bench_cfg2.err"; echo "bench cfg2 rc=$?" >> "$OUT/rc.txt"
timeout 600 python bench.py --form dual --no-cpu --also "" > "$OUT/bench_cfg2_dual.json" 2> "$OUT/bench_cfg2_dual.err"
timeout 600 python bench.py --workload cfg0 --steps 20000 --also "" > "$OUT/bench_cfg0.json" 2> "$OUT/bench_cfg0.err"
timeout 600 python bench.py --workload cfg1 --steps 20000 --also "" > "$OUT/bench_cfg1.json" 2> "$OUT/bench_cfg1.err"
timeout 900 python bench.py --workload cfg3 --steps 300 --warmup 20 > "$OUT/bench_cfg3.json" 2> "$OUT/bench_cfg3.err"
timeout 900 python bench.py --workload cfg4 --steps 20 > "$OUT/bench_cfg4.json" 2> "$OUT/bench_cfg4.err"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
python bench.py --steps 5 --warmup 3 --no-cpu --also "" --e2e-cap 0 > "$OUT/plain_cfg2.json" 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file "$OUT/launches_cfg2.csv" python bench.py --steps 5 --warmup 3 --no-cpu --also "" --e2e-cap 0 > "$OUT/ncu_l2.log" 2>&1
python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu --e2e-cap 0 > "$OUT/plain_cfg3.json" 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
    --log-file "$OUT/launches_cfg3.csv" python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu --e2e-cap 0 > "$OUT/ncu_l3.log" 2>&1
python bench.py --workload cfg4 --steps 2 --warmup 3 --no-cpu > "$OUT/plain_cfg4.json" 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
    --log-file "$OUT/launches_cfg4.csv" python bench.py --workload cfg4 --steps 2 --warmup 3 --no-cpu > "$OUT/ncu_l4.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemv_pieces|k_gemvT_rows|k_psd_wj32|k_syrk_dmma" -s 6 -c 5 \
  -o "$OUT/full_cfg2" python bench.py --steps 3 --warmup 3 --no-cpu --also "" > "$OUT/ncu_f2.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gtrd_tridiag|k_gtrd_vec|k_gtrd_back" -s 30 -c 3 \
  -o "$OUT/full_cfg3" python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu --e2e-cap 0 > "$OUT/ncu_f3.log" 2>&1
echo done >> "$OUT/rc.txt"
