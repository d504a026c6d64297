#!/usr/bin/env bash
# Round-2 final measurement pass: smoke, GPU tests, bench lines for every workload (+ the reference
# arm), ncu launch lists and full captures of the top kernels.  Output in gpurun_out/<tag>/.
set -u
TAG=${1:-s3final}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/rc.txt"
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/rc.txt"
timeout 900 python bench.py > "$OUT/bench_default.json" 2> "$OUT/bench_default.err"; echo "bench default rc=$?" >> "$OUT/rc.txt"
timeout 600 python bench.py --form dual --no-cpu --also "" > "$OUT/bench_cfg2_dual.json" 2> "$OUT/bench_cfg2_dual.err"
timeout 600 python bench.py --workload cfg0 --steps 20000 --also "" > "$OUT/bench_cfg0.json" 2> "$OUT/bench_cfg0.err"
timeout 600 python bench.py --workload cfg1 --steps 20000 --also "" > "$OUT/bench_cfg1.json" 2> "$OUT/bench_cfg1.err"
timeout 900 python bench.py --workload cfg3 --steps 300 --warmup 20 > "$OUT/bench_cfg3.json" 2> "$OUT/bench_cfg3.err"
timeout 900 python bench.py --workload cfg4 --steps 20 > "$OUT/bench_cfg4.json" 2> "$OUT/bench_cfg4.err"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
# launch lists (each after a clean plain run of the same command)
python bench.py --steps 5 --warmup 3 --no-cpu --also "" --e2e-cap 0 > "$OUT/plain_cfg2.json" 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file "$OUT/launches_cfg2.csv" python bench.py --steps 5 --warmup 3 --no-cpu --also "" --e2e-cap 0 > "$OUT/ncu_l2.log" 2>&1
python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu --e2e-cap 0 > "$OUT/plain_cfg3.json" 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
    --log-file "$OUT/launches_cfg3.csv" python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu --e2e-cap 0 > "$OUT/ncu_l3.log" 2>&1
python bench.py --workload cfg4 --steps 2 --warmup 3 --no-cpu > "$OUT/plain_cfg4.json" 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
    --log-file "$OUT/launches_cfg4.csv" python bench.py --workload cfg4 --steps 2 --warmup 3 --no-cpu > "$OUT/ncu_l4.log" 2>&1
python bench.py --workload cfg1 --steps 20 --warmup 3 --no-cpu --also "" --e2e-cap 0 > "$OUT/plain_cfg1.json" 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file "$OUT/launches_cfg1.csv" python bench.py --workload cfg1 --steps 20 --warmup 3 --no-cpu --also "" --e2e-cap 0 > "$OUT/ncu_l1.log" 2>&1
# full captures of the top kernels
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemv_pieces|k_gemvT_rows|k_psd_wj32" -s 6 -c 5 \
  -o "$OUT/full_cfg2" python bench.py --steps 3 --warmup 3 --no-cpu --also "" --e2e-cap 0 > "$OUT/ncu_f2.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gtrd" -s 20 -c 8 \
  -o "$OUT/full_cfg3" python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu --e2e-cap 0 > "$OUT/ncu_f3.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_trd_" -s 12 -c 12 \
  -o "$OUT/full_cfg4" python bench.py --workload cfg4 --steps 1 --warmup 3 --no-cpu > "$OUT/ncu_f4.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fused_iter" -s 10 -c 2 \
  -o "$OUT/full_cfg1" python bench.py --workload cfg1 --steps 20 --warmup 3 --no-cpu --also "" --e2e-cap 0 > "$OUT/ncu_f1.log" 2>&1
python tools/fused_probe2.py trace > "$OUT/fused_trace.log" 2>&1
# the reports are large (gpurun copies back <= 64 MiB): keep the raw-page CSV and the top SASS lines
for r in full_cfg1 full_cfg2 full_cfg3 full_cfg4; do
  if [ -f "$OUT/$r.ncu-rep" ]; then
    ncu -i "$OUT/$r.ncu-rep" --page raw --csv > "$OUT/${r}_raw.csv" 2>/dev/null
    ncu -i "$OUT/$r.ncu-rep" --page source --csv --print-source sass > "$OUT/${r}_sass.csv" 2>/dev/null
    gzip -f "$OUT/${r}_sass.csv"
    rm -f "$OUT/$r.ncu-rep"
  fi
done
du -sh "$OUT" >> "$OUT/rc.txt"
echo done >> "$OUT/rc.txt"
