#!/usr/bin/env bash
# Session-4 check: smoke, GPU suite, default bench line.  Output in gpurun_out/s4a/.
set -u
OUT=gpurun_out/s4a
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/rc.txt"
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/rc.txt"
timeout 900 python bench.py --workload cfg4 --steps 20 --no-cpu > "$OUT/bench_cfg4.json" 2> "$OUT/bench_cfg4.err"; echo "cfg4 rc=$?" >> "$OUT/rc.txt"
echo done >> "$OUT/rc.txt"
