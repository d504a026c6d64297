#!/usr/bin/env bash
OUT=gpurun_out/${1:-r2ac}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -q --timeout 300 -k "pinned or fused" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
timeout 300 python bench.py --workload cfg4 --steps 10 --no-cpu > $OUT/cfg4.json 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --also "" > $OUT/cfg2.json 2>&1
timeout 300 python bench.py --workload cfg1 --steps 20000 --also "" --no-cpu > $OUT/cfg1.json 2>&1
timeout 300 python bench.py --workload cfg0 --steps 20000 --also "" --no-cpu > $OUT/cfg0.json 2>&1
echo done >> $OUT/rc.txt
