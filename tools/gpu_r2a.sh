set -u
OUT=gpurun_out/r2a
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/rc.txt
timeout 1500 python -m pytest tests/test_gpu_boundary.py -x -q -m gpu > $OUT/boundary.log 2>&1; echo "boundary rc=$?" >> $OUT/rc.txt
timeout 2400 python -m pytest tests/test_gpu_parity.py -q -m gpu --durations=15 > $OUT/parity.log 2>&1; echo "parity rc=$?" >> $OUT/rc.txt
