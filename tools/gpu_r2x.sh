#!/usr/bin/env bash
# tier-stream priorities: cfg4 / cfg3 with the lead tier on a high-priority stream
OUT=gpurun_out/r2x; mkdir -p $OUT
for pr in 1 0; do for ns in 1 2; do
SDP_TIER_PRIO=$pr SDP_TIER_STREAMS=$ns timeout 300 python bench.py --workload cfg4 --steps 10 --no-cpu > $OUT/cfg4_p${pr}_s${ns}.json 2>&1
SDP_TIER_PRIO=$pr SDP_TIER_STREAMS=$ns timeout 300 python bench.py --workload cfg3 --steps 100 --warmup 20 --no-cpu --e2e-cap 0 > $OUT/cfg3_p${pr}_s${ns}.json 2>&1
done; done
echo done >> $OUT/rc.txt
