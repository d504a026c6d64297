set -u
OUT=gpurun_out/r2c
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_boundary.py -q -m gpu -x -k "sharded" -v > $OUT/sharded.log 2>&1; echo "sharded rc=$?" >> $OUT/rc.txt
for k in 65 100 200 400 630 800; do timeout 120 python tools/giant_one.py $k 2 3 >> $OUT/giant.log 2>&1; echo "k=$k rc=$?" >> $OUT/giant.log; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "gtrd or giant or cfg3" > $OUT/gtrd.log 2>&1; echo "gtrd rc=$?" >> $OUT/rc.txt
