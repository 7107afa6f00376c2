"""The paper's eigenvalue study with EXACT inner solves (test infrastructure: calls only oracle/
and workload/).

    python tests/scripts/spectrum_exact.py --dims 100,20 --out profiles/r02_spectrum_exact_100x20.json

PAPER.md "Behavior of Eigenvalues" (Fig. `evalues_plot`) shows the eigenvalues of
J M^-1 for CPR-AMG(1), CPR-AMG(2) and BF on the 2D 100 x 20 grid; its footnote says the
inverses of A_11, A_22 and the modified Schur complement were applied EXACTLY (Matlab
backslash), not by one AMG V-cycle.  The oracle reproduces that with one-level hierarchies
(max_coarse >= n: dense LU of A_ss, S~ and A_pp); the CPR first stage stays the block ILU(0)
(P:L172).  M^-1 is formed column by column from the oracle's preconditioner apply and the
spectrum of J M^-1 computed densely (numpy).  The same is done with the one-V-cycle inner solves
the solvers actually use (default AMG options), for comparison with the GPU study
(tools/spectrum.py).  Inputs: the C1 recipe on the paper's grid with gravity on and off (the
SPE10-derived Examples 1, 2 are not available).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from workload import make_system  # noqa: E402

NAMES = {0: "BF", 1: "CPR-AMG(1)", 2: "CPR-AMG(2)"}
BIG = 10 ** 7


def summary(lam):
    mag = np.abs(lam)
    return {"n_eig": int(lam.size), "min_abs": float(mag.min()), "frac_abs_lt_0.1": float(np.mean(mag < 0.1)),
            "max_abs_minus_1": float(np.max(np.abs(lam - 1))), "median_abs_minus_1": float(np.median(np.abs(lam - 1))),
            "re_range": [float(lam.real.min()), float(lam.real.max())], "im_max": float(np.abs(lam.imag).max())}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, default=1)
    p.add_argument("--dims", type=str, default="100,20")
    p.add_argument("--preconds", type=str, default="0,1,2")
    p.add_argument("--out", type=str, default=None)
    p.add_argument("--save", type=str, default=None, help="npz with the eigenvalues")
    a = p.parse_args()
    d = [int(x) for x in a.dims.split(",")] + [1]
    dims = tuple(d[:3])
    out = {"config": a.config, "dims": dims, "source": "oracle (plain C), dense numpy eig", "spectra": []}
    saved = {}
    for grav in (True, False):
        prob, J, rhs = make_system(a.config, dims=dims, gravity=grav)
        N = 2 * J.n
        D = J.to_dense()
        for pc in (int(q) for q in a.preconds.split(",")):
            for inner, mc in (("exact", BIG), ("one V-cycle", 64)):
                t0 = time.perf_counter()
                bf = oracle.BF(J, precond=pc, max_coarse=mc)
                Minv = np.empty((N, N))
                e = np.zeros(N)
                for j in range(N):
                    e[:] = 0.0
                    e[j] = 1.0
                    Minv[:, j] = bf.apply(e)
                lam = np.linalg.eigvals(D @ Minv)
                r = bf.gmres(rhs, tol=1e-8, restart=30, maxit=500)
                rec = {"precond": NAMES[pc], "inner_solves": inner, "gravity": grav, **summary(lam),
                       "gmres_iters_1e-8": r["iters"], "gmres_converged": r["converged"],
                       "seconds": time.perf_counter() - t0}
                out["spectra"].append(rec)
                saved[f"{NAMES[pc]} {inner}{'' if grav else ' (g=0)'}"] = lam
                print(json.dumps(rec), file=sys.stderr, flush=True)
    if a.save:
        np.savez_compressed(a.save, **saved)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
