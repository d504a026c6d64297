set -u
OUT=gpurun_out/r2n
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
SDP_TIER_STREAMS=1 timeout 600 python bench.py --workload cfg4 --steps 10 --no-cpu > $OUT/cfg4_s1.json 2> $OUT/cfg4_s1.err
timeout 600 python bench.py --workload cfg4 --steps 10 --no-cpu > $OUT/cfg4_s4.json 2> $OUT/cfg4_s4.err
SDP_TIER_STREAMS=1 timeout 600 python bench.py --workload cfg3 --steps 40 --no-cpu --e2e-cap 0 > $OUT/cfg3_s1.json 2> $OUT/cfg3_s1.err
timeout 600 python bench.py --workload cfg3 --steps 40 --no-cpu --e2e-cap 0 > $OUT/cfg3_s4.json 2> $OUT/cfg3_s4.err
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "batch or trd or giant_tier or gtrd" > $OUT/batch.log 2>&1; echo "batch rc=$?" >> $OUT/rc.txt
timeout 1200 python -m pytest tests/test_gpu_boundary.py -q -m gpu -k "forced_sparse or sensor_network_solve" > $OUT/sparse.log 2>&1; echo "sparse rc=$?" >> $OUT/rc.txt
