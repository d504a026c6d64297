#!/usr/bin/env bash
OUT=gpurun_out/${1:-r2y}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -q -x --timeout 300 -k "batch or iterates or fused or solve" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
python tools/fused_probe2.py trace > $OUT/trace.log 2>&1
timeout 300 python bench.py --workload cfg4 --steps 10 --no-cpu > $OUT/cfg4.json 2>&1
timeout 300 python bench.py --workload cfg3 --steps 100 --warmup 20 --no-cpu --e2e-cap 0 > $OUT/cfg3.json 2>&1
timeout 300 python bench.py --workload cfg0 --steps 20000 --also "" --no-cpu --e2e-cap 0 > $OUT/cfg0.json 2>&1
timeout 300 python bench.py --workload cfg1 --steps 20000 --also "" --no-cpu --e2e-cap 0 > $OUT/cfg1.json 2>&1
python tools/psd_batch_timing.py > $OUT/psd_tiers.txt 2>&1
echo done >> $OUT/rc.txt
