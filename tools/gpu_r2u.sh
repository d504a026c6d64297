#!/usr/bin/env bash
OUT=gpurun_out/r2u; mkdir -p $OUT
python tools/fused_probe2.py trace > $OUT/trace.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fused.py -q --timeout 300 > $OUT/pytest_fused.log 2>&1; echo "fused rc=$?" >> $OUT/rc.txt
python tools/fused_probe2.py long 0 > /dev/null 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fused -s 1 -c 1 -o $OUT/fused_cfg0 python tools/fused_probe2.py long 0 > $OUT/ncu0.log 2>&1
echo done >> $OUT/rc.txt
