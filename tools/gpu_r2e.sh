set -u
OUT=gpurun_out/r2e
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for k in 65 100 200 400 630 800; do timeout 120 python tools/giant_one.py $k 2 3 >> $OUT/giant.log 2>&1; echo "k=$k rc=$?" >> $OUT/giant.log; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launch_630.csv python tools/giant_one.py 630 1 1 > $OUT/ncu630.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "gtrd or giant or cfg3" > $OUT/gtrd.log 2>&1; echo "gtrd rc=$?" >> $OUT/rc.txt
timeout 300 python bench.py --workload cfg3 --steps 40 --no-cpu --e2e-cap 0 > $OUT/bench_cfg3.json 2> $OUT/bench_cfg3.err
