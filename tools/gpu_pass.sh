#!/usr/bin/env bash
# One GPU pass: parity tests, bench lines, ncu launch list and a full capture
# of the dominant kernel.  Usage (from the repo root, under gpurun):
#   bash tools/gpu_pass.sh [tag]
# Everything lands in gpurun_out/<tag>/.
set -u
TAG=${1:-pass}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > "$OUT/smi.txt" 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/rc.txt"
timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/rc.txt"
timeout 900 python bench.py > "$OUT/bench_cfg2.json" 2> "$OUT/bench_cfg2.err"; echo "bench cfg2 rc=$?" >> "$OUT/rc.txt"
timeout 600 python bench.py --form dual --no-cpu > "$OUT/bench_cfg2_dual.json" 2> "$OUT/bench_cfg2_dual.err"; echo "bench cfg2 dual rc=$?" >> "$OUT/rc.txt"
timeout 600 python bench.py --workload cfg1 --steps 20000 > "$OUT/bench_cfg1.json" 2> "$OUT/bench_cfg1.err"; echo "bench cfg1 rc=$?" >> "$OUT/rc.txt"
timeout 900 python bench.py --workload cfg3 --steps 100 > "$OUT/bench_cfg3.json" 2> "$OUT/bench_cfg3.err"; echo "bench cfg3 rc=$?" >> "$OUT/rc.txt"
timeout 900 python bench.py --workload cfg4 --steps 10 > "$OUT/bench_cfg4.json" 2> "$OUT/bench_cfg4.err"; echo "bench cfg4 rc=$?" >> "$OUT/rc.txt"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"; echo "bench ref rc=$?" >> "$OUT/rc.txt"
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$OUT/launches_cfg2.csv" python bench.py --steps 5 --warmup 3 --no-cpu > "$OUT/ncu_launch.log" 2>&1
  echo "ncu launches rc=$?" >> "$OUT/rc.txt"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_KERNEL:-k_gemv}" -c "${NCU_COUNT:-2}" \
    -o "$OUT/full_cfg2" python bench.py --steps 3 --warmup 3 --no-cpu > "$OUT/ncu_full.log" 2>&1
  echo "ncu full rc=$?" >> "$OUT/rc.txt"
fi
