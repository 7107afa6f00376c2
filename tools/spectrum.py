"""Eigenvalues of the preconditioned operator J M^-1 (the paper's
"Behavior of Eigenvalues" study, Fig. `evalues_plot`) for BF, CPR-AMG(1),
CPR-AMG(2) and the coupled AMG on a small 2D two-phase grid.

M^-1 is formed column by column from the GPU preconditioner apply (bf_apply_precond on unit
vectors, i.e. with the one-V-cycle inner solves actually used -- the paper's footnote used
exact inner solves), J M^-1 is formed densely on the host and its spectrum computed with
numpy.  GMRES convergence is governed by how far the spectrum stays from the origin
(`GMRES-bound`): the summary reports the smallest |lambda|, the fraction of
eigenvalues within 0.1 of the origin and the spread around 1.

    python tools/spectrum.py --dims 100,20 --config 1 > profiles/r01_spectrum.json
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1611_00127_b200 as bf
from workload import make_system

NAMES = {0: "BF", 1: "CPR-AMG(1)", 2: "CPR-AMG(2)", 3: "coupled AMG"}

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=1)
p.add_argument("--dims", type=str, default="100,20")
p.add_argument("--preconds", type=str, default="0,1,2,3")
p.add_argument("--save", type=str, default=None, help="npz with the eigenvalues")
a = p.parse_args()
d = [int(x) for x in a.dims.split(",")] + [1]
dims = tuple(d[:3])
out = {"config": a.config, "dims": dims, "spectra": []}
saved = {}
for grav in (True, False):
    prob, J, rhs = make_system(a.config, dims=dims, gravity=grav)
    N = 2 * J.n
    D = J.to_dense()
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    rp, ci, v = dev(J.row_ptr), dev(J.col_idx), dev(J.vals.reshape(-1))
    for pc in (int(q) for q in a.preconds.split(",")):
        s = bf.BFSolver(rp, ci, v, prob.dims, precond=pc)
        Minv = np.empty((N, N))
        e = torch.zeros(N, dtype=torch.float64, device="cuda")
        z = torch.empty(N, dtype=torch.float64, device="cuda")
        for j in range(N):
            e.zero_()
            e[j] = 1.0
            s.apply_precond(e, z)
            Minv[:, j] = z.cpu().numpy()
        rr = s.solve(dev(rhs), torch.zeros(N, dtype=torch.float64, device="cuda"), tol=1e-8, maxit=300)
        s.close()
        lam = np.linalg.eigvals(D @ Minv)
        mag = np.abs(lam)
        key = f"{NAMES[pc]}{'' if grav else ' (g=0)'}"
        saved[key] = lam
        out["spectra"].append({
            "precond": NAMES[pc], "gravity": grav, "n_eig": int(lam.size),
            "min_abs": float(mag.min()), "frac_abs_lt_0.1": float(np.mean(mag < 0.1)),
            "max_abs_minus_1": float(np.max(np.abs(lam - 1))), "median_abs_minus_1": float(np.median(np.abs(lam - 1))),
            "re_range": [float(lam.real.min()), float(lam.real.max())],
            "im_max": float(np.abs(lam.imag).max()),
            "gmres_iters_1e-8": rr["iters"], "gmres_converged": rr["converged"]})
        print(json.dumps(out["spectra"][-1]), file=sys.stderr, flush=True)
if a.save:
    np.savez_compressed(a.save, **saved)
print(json.dumps(out))
