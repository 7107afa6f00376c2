"""Small end-to-end runs of every solve path for compute-sanitizer (memcheck / racecheck /
synccheck, one tool per run):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_case.py

C1 (32x32) and a 20^3 C2 grid; for each: BF (l1-Jacobi and Chebyshev smoothers: split, S~,
cooperative PMIS, SpGEMMs, TMA-pipelined CSR kernels with mbarriers, DIA kernels, dense tail,
CUDA-graph apply, fused CGS2 reductions), CPR-AMG(2) (block ILU(0) factorization and the
sync-free pencil / value-flag sweeps), the coupled point AMG, bf_update, and a GMRES(40) solve
(CGS2 in 32-vector blocks).  Exits non-zero if any solve fails to converge where it should.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1611_00127_b200 as bf
from workload import make_system

dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
ok = True
for cfg, dims in ((1, None), (2, (20, 20, 20))):
    prob, J, rhs = make_system(cfg, dims=dims)
    rp, ci, v, b = dev(J.row_ptr), dev(J.col_idx), dev(J.vals.reshape(-1)), dev(rhs)
    for name, opts, restart, expect in (("BF l1", dict(), 30, True), ("BF cheb", dict(smoother=1, cheb_lo=0.1), 30, True),
                                         ("BF m=40", dict(), 40, True), ("CPR-AMG(2)", dict(precond=2), 30, True),
                                         ("CPR-AMG(1) flags", dict(precond=1), 30, True),
                                         ("coupled AMG", dict(precond=3), 30, False)):
        s = bf.BFSolver(rp, ci, v, prob.dims, **opts)
        x = torch.zeros(2 * J.n, dtype=torch.float64, device="cuda")
        r = s.solve(b, x, tol=1e-8, restart=restart, maxit=150 if expect else 20)
        if name == "BF l1":
            s.update(v)  # setup reuse on the same values
            x.zero_()
            r2 = s.solve(b, x, tol=1e-8, restart=restart, maxit=150)
            ok &= r2["converged"]
        torch.cuda.synchronize()
        print(f"C{cfg} {prob.dims} {name}: iters {r['iters']} converged {r['converged']} relres {r['relres']:.2e}",
              flush=True)
        if expect and not r["converged"]:
            ok = False
        s.close()
torch.cuda.synchronize()
print("sanitize_case:", "OK" if ok else "FAILED")
sys.exit(0 if ok else 1)
