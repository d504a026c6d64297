#!/usr/bin/env bash
OUT=gpurun_out/${1:-r2z}; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_parity.py -q -x --timeout 600 -k "not slow" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
SDP_SETUP_TRACE=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --also "" > $OUT/cfg2.json 2> $OUT/cfg2.err
echo done >> $OUT/rc.txt
