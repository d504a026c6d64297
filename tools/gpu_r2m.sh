set -u
OUT=gpurun_out/r2m
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_boundary.py -q -m gpu -k "sensor or forced_sparse or sharded" > $OUT/sparse.log 2>&1; echo "sparse rc=$?" >> $OUT/rc.txt
SDP_SETUP_TRACE=1 timeout 300 python -c "
import sys, time; sys.path.insert(0,'.')
import torch; torch.zeros(1).cuda()
import paper_1609_06068_b200 as L, sdp_inputs as gen
p = gen.sensor_network(2000, 0.032, seed=7)
t=time.time(); s = L.Solver(p, form='primal', rho=1.0); print('setup', time.time()-t, s.info()['s_factor'], s.info()['nnz_l'])
torch.cuda.synchronize(); t=time.time(); s.step(200); torch.cuda.synchronize(); print('it/s', 200/(time.time()-t))
" > $OUT/sensor_setup.log 2>&1
SDP_SPARSE_S=0 SDP_SETUP_TRACE=1 timeout 300 python -c "
import sys, time; sys.path.insert(0,'.')
import torch; torch.zeros(1).cuda()
import paper_1609_06068_b200 as L, sdp_inputs as gen
p = gen.sensor_network(2000, 0.032, seed=7)
t=time.time(); s = L.Solver(p, form='primal', rho=1.0); print('setup dense', time.time()-t, s.info()['s_factor'])
" >> $OUT/sensor_setup.log 2>&1
