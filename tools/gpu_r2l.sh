set -u
OUT=gpurun_out/r2l
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_boundary.py -q -m gpu -k "sharded" > $OUT/sharded.log 2>&1; echo "sharded rc=$?" >> $OUT/rc.txt
python tools/sanitize_case.py batch > $OUT/plain_batch.log 2>&1 && timeout 900 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_case.py batch > $OUT/racecheck_batch.log 2>&1; echo "race batch rc=$?" >> $OUT/rc.txt
