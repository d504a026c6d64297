#!/usr/bin/env bash
# full GPU suite + cfg3 giant-tier full capture
set -u
OUT=gpurun_out/r2q; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu --e2e-cap 0 > $OUT/plain_cfg3.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gtrd" -s 20 -c 8 \
  -o $OUT/full_cfg3 python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu --e2e-cap 0 > $OUT/ncu_f3.log 2>&1
echo "done" >> $OUT/rc.txt
