"""Config 5 (256x256x128, 16.8M DOF): the 5 Jacobians of 5 undamped Newton steps of one
implicit time step, each solved on the GPU (GMRES(30), tol 1e-8, maxit capped), with
(a) a full bf_setup per Jacobian and (b) bf_setup once + bf_update (setup reuse, R16).
Newton states come from mode (a)'s solves (reading Q18); both modes are timed on the same
J(u_k).  Prints one JSON line."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1611_00127_b200 as bf
from workload import newton_sequence

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=5)
p.add_argument("--dims", type=str, default=None)
p.add_argument("--steps", type=int, default=5)
p.add_argument("--maxit", type=int, default=2500)
p.add_argument("--restart", type=int, default=200)
p.add_argument("--opts", type=str, default="", help="bf_options, e.g. cheb_degree=3,cheb_lo=0.05")
a = p.parse_args()
_val = lambda v: float(v) if ("." in v or "e" in v) else int(v)
OPT = bf.bf_default_options(**{k: _val(v) for k, v in (kv.split("=") for kv in a.opts.split(",") if kv)})
dims = tuple(int(x) for x in a.dims.split(",")) if a.dims else None
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
ev = lambda: torch.cuda.Event(enable_timing=True)
rec = []
reuse = {"h": None}


def solve(k, J, rhs):
    rp, ci, v, b = dev(J.row_ptr), dev(J.col_idx), dev(J.vals.reshape(-1)), dev(rhs)
    out = {"k": k}
    # (a) full setup
    x = torch.zeros(2 * J.n, dtype=torch.float64, device="cuda")
    e0, e1, e2 = ev(), ev(), ev()
    e0.record()
    h = bf.bf_setup(rp, ci, v, dims_k, opt=OPT)
    e1.record()
    r = bf.bf_solve(h, b, x, 1e-8, a.restart, a.maxit)
    e2.record()
    torch.cuda.synchronize()
    out.update(full_setup_ms=e0.elapsed_time(e1), full_solve_ms=e1.elapsed_time(e2), full_iters=r["iters"],
               full_relres=r["relres"], full_converged=r["converged"])
    bf.bf_destroy(h)
    # (b) reuse: setup once at k = 0, bf_update afterwards
    x2 = torch.zeros(2 * J.n, dtype=torch.float64, device="cuda")
    e0, e1, e2 = ev(), ev(), ev()
    e0.record()
    if reuse["h"] is None:
        reuse["h"] = bf.bf_setup(rp, ci, v, dims_k, opt=OPT)
    else:
        bf.bf_update(reuse["h"], v)
    e1.record()
    r2 = bf.bf_solve(reuse["h"], b, x2, 1e-8, a.restart, a.maxit)
    e2.record()
    torch.cuda.synchronize()
    out.update(reuse_setup_ms=e0.elapsed_time(e1), reuse_solve_ms=e1.elapsed_time(e2), reuse_iters=r2["iters"],
               reuse_relres=r2["relres"], reuse_converged=r2["converged"])
    rec.append(out)
    print(json.dumps(out), file=sys.stderr, flush=True)
    return x.cpu().numpy()


dims_k = None
t0 = time.perf_counter()
fnorms = []
for k, prob, J, rhs, fn in newton_sequence(a.config, a.steps, solve, dims=dims):
    dims_k = prob.dims
    fnorms.append(fn)
tot = lambda key: sum(r[key] for r in rec)
print(json.dumps({"config": a.config, "dims": dims_k, "steps": a.steps, "dof": 2 * prob.n, "restart": a.restart,
                  "opts": a.opts, "newton_F_norms": fnorms,
                  "full_total_ms": tot("full_setup_ms") + tot("full_solve_ms"),
                  "reuse_total_ms": tot("reuse_setup_ms") + tot("reuse_solve_ms"),
                  "full_setup_ms": tot("full_setup_ms"), "reuse_setup_ms": tot("reuse_setup_ms"),
                  "full_iters": [r["full_iters"] for r in rec], "reuse_iters": [r["reuse_iters"] for r in rec],
                  "full_relres": [r["full_relres"] for r in rec], "reuse_relres": [r["reuse_relres"] for r in rec],
                  "full_converged": [r["full_converged"] for r in rec], "reuse_converged": [r["reuse_converged"] for r in rec],
                  "wall_s": time.perf_counter() - t0}))
