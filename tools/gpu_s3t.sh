#!/usr/bin/env bash
# root-free QL A/B: trd / batch tests with it on, bucket timing on / off, launch list with it on
OUT=gpurun_out/${1:-s3t}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
SDP_TRD_QLPWK=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "trd or batch" > $OUT/pytest_trd_pwk.log 2>&1; echo "pytest pwk rc=$?" >> $OUT/rc.txt
timeout 300 python tools/psd_batch_timing.py 16,32,64 > $OUT/timing.txt 2>&1
SDP_TRD_QLPWK=1 timeout 300 python tools/psd_batch_timing.py 16,32,64 > $OUT/timing_pwk.txt 2>&1
SDP_TRD_QLPWK=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_pwk.csv python tools/psd_batch_timing.py 16,32,64 > $OUT/ncu_l.log 2>&1
echo done >> $OUT/rc.txt
