"""Why the later C5 Newton Jacobians do not converge: builds u_1 from the
GPU solve of J(u_0) exactly as tools/newton_c5.py does (saturation chop, reading R17), then on
J(u_1) reports the state (saturations at the bounds, the pressure update, the spread of the
A_ss and A_pp diagonals) and GMRES(m) to 1e-8 with several preconditioners: BF (default R22,
Chebyshev on both hierarchies, l1-Jacobi on both) and CPR-AMG(2) (global ILU(0) first stage).
If every preconditioner stalls, the difficulty is the Jacobian, not the BF apply.

    python tools/c5_newton_diag.py [--dims 128,128,64] [--restart 200] [--maxit 1500]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1611_00127_b200 as bf
from workload import newton_sequence

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=5)
p.add_argument("--dims", type=str, default=None)
p.add_argument("--restart", type=int, default=200)
p.add_argument("--maxit", type=int, default=1500)
a = p.parse_args()
dims = tuple(int(x) for x in a.dims.split(",")) if a.dims else None
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
PRECS = [("BF default (R22)", {}), ("BF Chebyshev both", dict(smoother_p=-1, cheb_lo=0.15)),
         ("BF l1 both", dict(smoother=0)), ("CPR-AMG(2)", dict(precond=2))]


def run(J, rhs, dims_k, opts):
    rp, ci, v, b = dev(J.row_ptr), dev(J.col_idx), dev(J.vals.reshape(-1)), dev(rhs)
    x = torch.zeros(2 * J.n, dtype=torch.float64, device="cuda")
    h = bf.bf_setup(rp, ci, v, dims_k, opt=bf.bf_default_options(**opts))
    try:
        r = bf.bf_solve(h, b, x, 1e-8, a.restart, a.maxit)
    except bf.BFError as e:
        bf.bf_destroy(h)
        return {"error": str(e)}, None
    bf.bf_destroy(h)
    return {"iters": r["iters"], "converged": r["converged"], "relres": r["relres"],
            "hist_every_100": [float(t) for t in r["hist"][::100]]}, x.cpu().numpy()


def stats(J, sn, p0, p):
    blocks = J.vals
    diag = np.array([blocks[J.row_ptr[i] + np.searchsorted(J.col_idx[J.row_ptr[i]:J.row_ptr[i + 1]], i)]
                     for i in range(0, J.n, max(1, J.n // 200000))])
    app, ass = diag[:, 0, 0], diag[:, 1, 1]
    return {"sn_at_0": float(np.mean(sn <= 0.0)), "sn_at_1": float(np.mean(sn >= 1.0)),
            "sn_min": float(sn.min()), "sn_max": float(sn.max()),
            "dp_max_abs": float(np.abs(p - p0).max()), "p_range": [float(p.min()), float(p.max())],
            "A_pp_diag_range(sample)": [float(app.min()), float(app.max())],
            "A_ss_diag_range(sample)": [float(ass.min()), float(ass.max())]}


out = {"config": a.config, "restart": a.restart, "maxit": a.maxit, "jacobians": []}
state = {}


def solve(k, J, rhs):
    dims_k = state["dims"]
    rec = {"k": k, "F_norm": float(np.linalg.norm(rhs))}
    if k >= 1:
        rec["state"] = stats(J, state["sn"], state["p0"], state["p"])
        for name, opts in PRECS:
            rec[name] = run(J, rhs, dims_k, opts)[0]
            print(json.dumps({"k": k, name: rec[name]}), file=sys.stderr, flush=True)
    res, x = run(J, rhs, dims_k, {})
    rec.setdefault("BF default (R22)", res)
    out["jacobians"].append(rec)
    return x if x is not None else np.zeros(2 * J.n)


gen = newton_sequence(a.config, 2, solve, dims=dims)
for k, prob, J, rhs, fn in gen:
    state["dims"] = prob.dims
    if k == 0:
        state["p0"] = prob.p_old.copy()
    # the generator's current state is reconstructed from J's inputs: track it through the updates
    state["p"] = getattr(prob, "_p_cur", prob.p_old)
    state["sn"] = getattr(prob, "_sn_cur", prob.sn_old)
print(json.dumps(out))
