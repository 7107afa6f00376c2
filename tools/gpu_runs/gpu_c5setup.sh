set -x
BF_VERBOSE=1 timeout 400 python -c "
import time, numpy as np, torch, sys
sys.path.insert(0,'.')
from workload import make_system
import paper_1611_00127_b200 as bf
t=time.time(); prob,J,rhs=make_system(5); print('make', time.time()-t, flush=True)
dev=lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
rp,ci,v=dev(J.row_ptr),dev(J.col_idx),dev(J.vals.reshape(-1)); torch.cuda.synchronize(); print('copied', time.time()-t, flush=True)
s=bf.BFSolver(rp,ci,v,prob.dims); torch.cuda.synchronize(); print('setup', time.time()-t, flush=True)
x=torch.zeros(2*J.n,dtype=torch.float64,device='cuda')
r=s.solve(dev(rhs),x,tol=0.0,maxit=5); print('solve5', time.time()-t, r['relres'], flush=True)
" > gpurun_out/c5setup.txt 2>&1
tail -40 gpurun_out/c5setup.txt
