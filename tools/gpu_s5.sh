#!/usr/bin/env bash
# Session-5 check of the restored tree: smoke, GPU suite, the default bench line and the reference arm.  Output in gpurun_out/s5/.
set -u
OUT=gpurun_out/s5
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/rc.txt"
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/rc.txt"
timeout 600 python bench.py > "$OUT/bench_default.json" 2> "$OUT/bench_default.err"; echo "default rc=$?" >> "$OUT/rc.txt"
timeout 300 python bench.py --impl reference > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"; echo "ref rc=$?" >> "$OUT/rc.txt"
echo done >> "$OUT/rc.txt"
