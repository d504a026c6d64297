#!/usr/bin/env bash
OUT=gpurun_out/${1:-r2aa}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_schur.py -q --timeout 300 > $OUT/pytest_schur.log 2>&1; echo "schur rc=$?" >> $OUT/rc.txt
timeout 900 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_parity.py -q --timeout 300 -k "ill or error or sensor or sparse or solve" > $OUT/pytest_b.log 2>&1; echo "b rc=$?" >> $OUT/rc.txt
SDP_SETUP_TRACE=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --also "" > $OUT/cfg2.json 2> $OUT/cfg2.err
echo done >> $OUT/rc.txt
