#!/usr/bin/env bash
# cfg4 A/B: tier streams 1..4
OUT=gpurun_out/${1:-s3m}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for t in 1 2 3 4; do SDP_TIER_STREAMS=$t timeout 600 python bench.py --workload cfg4 --steps 20 --no-cpu > $OUT/cfg4_ts$t.json 2> $OUT/cfg4_ts$t.err; done
echo done >> $OUT/rc.txt
