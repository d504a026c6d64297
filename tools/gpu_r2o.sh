set -u
OUT=gpurun_out/r2o
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for k in 200 400 630; do timeout 120 python tools/giant_one.py $k 1 5 >> $OUT/giant.log 2>&1; done
SDP_GTRD_DEBUG=2 timeout 120 python tools/giant_one.py 630 1 1 > $OUT/dbg630.log 2>&1
timeout 600 python bench.py --workload cfg3 --steps 40 --no-cpu --e2e-cap 0 > $OUT/cfg3.json 2> $OUT/cfg3.err
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "gtrd or giant or cfg3" > $OUT/gtrd.log 2>&1; echo "gtrd rc=$?" >> $OUT/rc.txt
