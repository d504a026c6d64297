set -u
OUT=gpurun_out/r2d
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_boundary.py -q -m gpu -k "sharded" > $OUT/sharded.log 2>&1; echo "sharded rc=$?" >> $OUT/rc.txt
python tools/giant_one.py 630 1 3 > $OUT/g630.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launch_630.csv python tools/giant_one.py 630 1 1 > $OUT/ncu630.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launch_200.csv python tools/giant_one.py 200 8 1 > $OUT/ncu200.log 2>&1
