#!/usr/bin/env bash
OUT=gpurun_out/r2t; mkdir -p $OUT
python tools/fused_probe2.py trace > $OUT/trace.log 2>&1
SDP_FUSED=0 python tools/fused_probe2.py trace > $OUT/trace_unfused.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x --timeout 300 > $OUT/pytest_fused.log 2>&1; echo "fused rc=$?" >> $OUT/rc.txt
timeout 300 python bench.py --workload cfg0 --steps 20000 --also "" --no-cpu --e2e-cap 0 > $OUT/bench_cfg0.json 2>&1
timeout 300 python bench.py --workload cfg1 --steps 20000 --also "" --no-cpu --e2e-cap 0 > $OUT/bench_cfg1.json 2>&1
echo done >> $OUT/rc.txt
