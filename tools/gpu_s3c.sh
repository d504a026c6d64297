#!/usr/bin/env bash
# QL tier: trd / batch tests, k = 32 / 64 bucket timing, launch list, full capture of the k = 64 kernels.
OUT=gpurun_out/${1:-s3c}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "trd or batch" > $OUT/pytest_trd.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
timeout 300 python tools/psd_batch_timing.py 32,64 > $OUT/timing.txt 2>&1
SDP_TRD_QLFUSED=0 timeout 300 python tools/psd_batch_timing.py 32,64 > $OUT/timing_unfused.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
    --log-file $OUT/launches.csv python tools/psd_batch_timing.py 32,64 > $OUT/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_trd_" -c 4 -o $OUT/full_k64 python tools/psd_batch_timing.py 64 > $OUT/ncu_f.log 2>&1
if [ -f $OUT/full_k64.ncu-rep ]; then
  ncu -i $OUT/full_k64.ncu-rep --page raw --csv > $OUT/full_k64_raw.csv 2>/dev/null
  ncu -i $OUT/full_k64.ncu-rep --page source --csv --print-source sass > $OUT/full_k64_sass.csv 2>/dev/null
  gzip -f $OUT/full_k64_sass.csv; rm -f $OUT/full_k64.ncu-rep
fi
echo done >> $OUT/rc.txt
