#!/usr/bin/env bash
OUT=gpurun_out/${1:-r2ad}; mkdir -p $OUT
for c in 2 4 8 16; do SDP_PSD_PIPE_CHUNKS=$c timeout 300 python bench.py --workload cfg4 --steps 3 --no-cpu > $OUT/cfg4_c$c.json 2>&1; done
echo done >> $OUT/rc.txt
