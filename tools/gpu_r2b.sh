set -u
OUT=gpurun_out/r2b
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_boundary.py -q -m gpu --durations=10 > $OUT/boundary.log 2>&1; echo "boundary rc=$?" >> $OUT/rc.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/rc.txt
SDP_GTRD_DEBUG=2 timeout 300 python tools/giant_one.py 630 1 3 > $OUT/giant630_dbg.log 2>&1
timeout 300 python tools/giant_one.py 630 1 5 > $OUT/giant630.log 2>&1
timeout 300 python tools/giant_one.py 200 8 5 >> $OUT/giant630.log 2>&1
timeout 300 python tools/giant_one.py 100 16 5 >> $OUT/giant630.log 2>&1
