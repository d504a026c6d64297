#!/usr/bin/env bash
# Session-3 check of HEAD: smoke, GPU suite, short bench lines for the latency and batch workloads.
OUT=gpurun_out/${1:-s3a}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/rc.txt
timeout 600 python bench.py --workload cfg0 --steps 20000 --also "" --no-cpu > $OUT/cfg0.json 2> $OUT/cfg0.err
timeout 600 python bench.py --workload cfg1 --steps 20000 --also "" --no-cpu > $OUT/cfg1.json 2> $OUT/cfg1.err
timeout 600 python bench.py --workload cfg4 --steps 20 --no-cpu > $OUT/cfg4.json 2> $OUT/cfg4.err
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
echo done >> $OUT/rc.txt
