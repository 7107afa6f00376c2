"""Attainable-accuracy check on C5: after the GPU solve, compare the relative residual floor with
eps * || |J| |x| || / ||b|| (the rounding floor of the residual b - J x evaluated in fp64)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1611_00127_b200 as bf
from workload import make_system

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
prob, J, rhs = make_system(cfg)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
s = bf.BFSolver(dev(J.row_ptr), dev(J.col_idx), dev(J.vals.reshape(-1)), prob.dims)
x = torch.zeros(2 * J.n, dtype=torch.float64, device="cuda")
r = s.solve(dev(rhs), x, tol=1e-8, maxit=900)
xh = x.cpu().numpy()
A = J.to_scipy()
absJx = abs(A) @ np.abs(xh)
res = rhs - A @ xh
eps = np.finfo(np.float64).eps
print({"config": cfg, "iters": r["iters"], "relres": r["relres"],
       "floor_eps_absJ_absx_over_b": float(eps * np.linalg.norm(absJx) / np.linalg.norm(rhs)),
       "componentwise_backward_err": float(np.max(np.abs(res) / (absJx + np.abs(rhs)))),
       "norm_x_p": float(np.linalg.norm(xh[0::2])), "norm_x_s": float(np.linalg.norm(xh[1::2])),
       "norm_b_w": float(np.linalg.norm(rhs[0::2])), "norm_b_n": float(np.linalg.norm(rhs[1::2])),
       "relres_w_rows": float(np.linalg.norm(res[0::2]) / np.linalg.norm(rhs)),
       "relres_n_rows": float(np.linalg.norm(res[1::2]) / np.linalg.norm(rhs))}, flush=True)
