#!/usr/bin/env bash
OUT=gpurun_out/${1:-r2ab}; mkdir -p $OUT
for sp in 1 2 4 8; do for ns in 2 4; do
  if [ $sp = 1 ] && [ $ns = 4 ]; then continue; fi
  SDP_TRD_SPLIT=$sp SDP_TRD_SPLIT_STREAMS=$ns timeout 300 python bench.py --workload cfg4 --steps 10 --no-cpu > $OUT/cfg4_s${sp}_n${ns}.json 2>&1
done; done
SDP_TRD_SPLIT=4 timeout 300 python tools/psd_batch_timing.py > $OUT/tiers_s4.txt 2>&1
timeout 300 python tools/psd_batch_timing.py > $OUT/tiers_s1.txt 2>&1
echo done >> $OUT/rc.txt
