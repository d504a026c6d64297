#!/usr/bin/env bash
# flakiness probe of the cfg2 loopback-sharded test: default tier streams vs 1
OUT=gpurun_out/${1:-s3r}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for i in 1 2 3 4; do timeout 600 python -m pytest tests/test_gpu_boundary.py -q -k "sharded_loopback_cfg2 and primal" > $OUT/def_$i.log 2>&1; echo "def $i rc=$?" >> $OUT/rc.txt; done
for i in 1 2 3; do SDP_TIER_STREAMS=1 timeout 600 python -m pytest tests/test_gpu_boundary.py -q -k "sharded_loopback_cfg2 and primal" > $OUT/ts1_$i.log 2>&1; echo "ts1 $i rc=$?" >> $OUT/rc.txt; done
echo done >> $OUT/rc.txt
