#!/usr/bin/env bash
OUT=gpurun_out/r2s; mkdir -p $OUT
python tools/fused_probe2.py trace > $OUT/trace.log 2>&1
for c in 0 1; do for f in 1 0; do
python tools/fused_probe2.py steps $c $f > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --cache-control all --clock-control none --csv --log-file $OUT/ncu_c${c}_f${f}.csv python tools/fused_probe2.py steps $c $f > $OUT/ncu_c${c}_f${f}.log 2>&1
done; done
echo done > $OUT/rc.txt
