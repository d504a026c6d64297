#!/usr/bin/env bash
# KP = 8 QL tier: trd / batch tests, k = 8 bucket on / off, cfg4, cfg3 (small cliques) on / off
OUT=gpurun_out/${1:-s3u}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "trd or batch" > $OUT/pytest_trd.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
timeout 300 python tools/psd_batch_timing.py 8,16 > $OUT/timing.txt 2>&1
SDP_TRD8=0 timeout 300 python tools/psd_batch_timing.py 8 > $OUT/timing_rv8.txt 2>&1
timeout 600 python bench.py --workload cfg4 --steps 20 --no-cpu > $OUT/cfg4.json 2> $OUT/cfg4.err
SDP_TRD8=0 timeout 600 python bench.py --workload cfg4 --steps 20 --no-cpu > $OUT/cfg4_rv8.json 2> $OUT/cfg4_rv8.err
timeout 600 python bench.py --workload cfg3 --steps 100 --warmup 20 --no-cpu --e2e-cap 0 > $OUT/cfg3.json 2> $OUT/cfg3.err
SDP_TRD8=0 timeout 600 python bench.py --workload cfg3 --steps 100 --warmup 20 --no-cpu --e2e-cap 0 > $OUT/cfg3_rv8.json 2> $OUT/cfg3_rv8.err
echo done >> $OUT/rc.txt
