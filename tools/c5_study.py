"""C5 (256x256x128, 16.8M DOF) convergence study: GMRES(m) with restarts
beyond 32 (the CGS2 passes now run in 32-vector blocks) and the Chebyshev smoother on J(u_0),
BF preconditioner.  One JSON line per (restart, options) with the residual history every 100
iterations, setup / solve times (CUDA events) and the device memory of the handle.

    python tools/c5_study.py --restarts 30,100,200 --maxit 3000 --opts "nu_pre=1;smoother=1,cheb_lo=0.1"
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

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=5)
p.add_argument("--dims", type=str, default=None)
p.add_argument("--restarts", type=str, default="30,100,200")
p.add_argument("--maxit", type=int, default=3000)
p.add_argument("--tol", type=float, default=1e-8)
p.add_argument("--opts", type=str, default="nu_pre=1")
a = p.parse_args()
dims = tuple(int(x) for x in a.dims.split(",")) if a.dims else None
prob, J, rhs = make_system(a.config, dims=dims)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
rp, ci, v, b = dev(J.row_ptr), dev(J.col_idx), dev(J.vals.reshape(-1)), dev(rhs)


def parse(grp):
    val = lambda s: float(s) if ("." in s or "e" in s) else int(s)
    return {k: val(x) for k, x in (kv.split("=") for kv in grp.split(",") if kv)}


for opts in (parse(g) for g in a.opts.split(";")):
    for m in (int(r) for r in a.restarts.split(",")):
        o = bf.bf_default_options(**opts)
        x = torch.zeros(2 * J.n, dtype=torch.float64, device="cuda")
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        torch.cuda.synchronize()
        e[0].record()
        h = bf.bf_setup(rp, ci, v, prob.dims, opt=o)
        e[1].record()
        try:
            r = bf.bf_solve(h, b, x, a.tol, m, a.maxit)
            e[2].record()
            torch.cuda.synchronize()
            rec = {"config": a.config, "dims": prob.dims, "restart": m, "opts": opts, "iters": r["iters"],
                   "converged": r["converged"], "relres": r["relres"], "setup_ms": e[0].elapsed_time(e[1]),
                   "solve_ms": e[1].elapsed_time(e[2]), "device_GB": bf.bf_device_bytes(h) / 1e9,
                   "hist_every_100": [float(t) for t in r["hist"][::100]]}
        except Exception as ex:
            rec = {"config": a.config, "restart": m, "opts": opts, "error": str(ex)}
        bf.bf_destroy(h)
        print(json.dumps(rec), flush=True)
