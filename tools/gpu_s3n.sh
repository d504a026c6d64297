#!/usr/bin/env bash
# tier streams 1 vs 2 on cfg3 (cfg4 measured in s3m)
OUT=gpurun_out/${1:-s3n}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for t in 1 2; do SDP_TIER_STREAMS=$t timeout 600 python bench.py --workload cfg3 --steps 100 --warmup 20 --no-cpu --e2e-cap 0 > $OUT/cfg3_ts$t.json 2> $OUT/cfg3_ts$t.err; done
for t in 1 2; do SDP_TIER_STREAMS=$t timeout 600 python bench.py --workload cfg1 --steps 5000 --no-cpu --also "" --e2e-cap 0 > $OUT/cfg1_ts$t.json 2> $OUT/cfg1_ts$t.err; done
echo done >> $OUT/rc.txt
