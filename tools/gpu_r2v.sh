#!/usr/bin/env bash
OUT=gpurun_out/r2v; mkdir -p $OUT
for c in 0 1; do
python tools/fused_probe2.py long $c 0 > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file $OUT/warm_c${c}_unfused.csv python tools/fused_probe2.py long $c 0 > $OUT/l$c.log 2>&1
done
echo done >> $OUT/rc.txt
