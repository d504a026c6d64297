#!/usr/bin/env bash
# fused small-problem iteration: tests + cfg0/cfg1 bench lines
set -u
OUT=gpurun_out/r2r; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x --timeout 300 > $OUT/pytest_fused.log 2>&1; echo "fused rc=$?" >> $OUT/rc.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "cfg0 or cfg1 or arrow or trace1 or theta5 or determinism or set_rho or affine or solve" > $OUT/pytest_parity.log 2>&1; echo "parity rc=$?" >> $OUT/rc.txt
timeout 300 python bench.py --workload cfg0 --steps 20000 --also "" > $OUT/bench_cfg0.json 2> $OUT/bench_cfg0.err
timeout 300 python bench.py --workload cfg1 --steps 20000 --also "" > $OUT/bench_cfg1.json 2> $OUT/bench_cfg1.err
timeout 300 python bench.py --workload cfg1 --form dual --steps 20000 --also "" --no-cpu > $OUT/bench_cfg1_dual.json 2> $OUT/bench_cfg1_dual.err
for c in 1 8 37 74 148; do SDP_FUSED_CTAS=$c timeout 300 python bench.py --workload cfg1 --steps 5000 --also "" --no-cpu --e2e-cap 0 > $OUT/bench_cfg1_c$c.json 2>&1; done
SDP_FUSED=0 timeout 300 python bench.py --workload cfg1 --steps 5000 --also "" --no-cpu --e2e-cap 0 > $OUT/bench_cfg1_unfused.json 2>&1
echo done >> $OUT/rc.txt
