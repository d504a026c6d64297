#!/usr/bin/env bash
# KP = 16 QL tier: trd / batch tests, bucket timing with the tier on / off, cfg4 bench, launch list.
OUT=gpurun_out/${1:-s3e}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "trd or batch" > $OUT/pytest_trd.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
timeout 300 python tools/psd_batch_timing.py 16,32,64 > $OUT/timing.txt 2>&1
SDP_TRD_SPLIT=0 timeout 300 python tools/psd_batch_timing.py 16,32,64 > $OUT/timing_nosplit.txt 2>&1
timeout 600 python bench.py --workload cfg4 --steps 20 --no-cpu > $OUT/cfg4.json 2> $OUT/cfg4.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
    --log-file $OUT/launches.csv python tools/psd_batch_timing.py 16,32,64 > $OUT/ncu_l.log 2>&1
echo done >> $OUT/rc.txt
