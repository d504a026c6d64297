set -u
OUT=gpurun_out/r2j
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
SDP_SETUP_TRACE=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import paper_1609_06068_b200 as L, sdp_inputs as gen, time
p = gen.config(2)
t=time.time(); s = L.Solver(p, form='primal', rho=10.0); print('setup wall', time.time()-t, 'info', s.info()['setup_s'])
p3 = gen.config(3)
t=time.time(); s3 = L.Solver(p3, form='primal', rho=0.1); print('setup3 wall', time.time()-t)
" > $OUT/setup_trace.log 2>&1
timeout 900 python -m pytest tests/test_gpu_boundary.py -q -m gpu > $OUT/boundary.log 2>&1; echo "boundary rc=$?" >> $OUT/rc.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "solve_objective or iterates_after_50 or checkpoint" > $OUT/parity_sub.log 2>&1; echo "parity rc=$?" >> $OUT/rc.txt
timeout 900 python bench.py --also "" > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/rc.txt
