set -u
OUT=gpurun_out/r2f
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
SDP_GTRD_DEBUG=3 timeout 120 python tools/giant_one.py 630 1 1 > $OUT/dbg630.log 2>&1
SDP_GTRD_DEBUG=3 timeout 120 python tools/giant_one.py 200 1 1 > $OUT/dbg200.log 2>&1
