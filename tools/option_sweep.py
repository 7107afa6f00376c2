"""Iterations and time-to-solution of the GPU solver for several option sets (one config)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1611_00127_b200 as bf
from workload import make_system

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=3)
p.add_argument("--dims", type=str, default=None)
p.add_argument("--maxit", type=int, default=1500)
p.add_argument("--sets", type=str, default="all")
p.add_argument("--opts", type=str, default=None,
               help="';'-separated option sets, e.g. 'smoother=1,cheb_lo=0.1;nu_pre=2,nu_post=2'")
p.add_argument("--restart", type=int, default=30)
a = p.parse_args()
dims = tuple(int(x) for x in a.dims.split(",")) if a.dims else None
prob, J, rhs = make_system(a.config, dims=dims)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
rp, ci, v, b = dev(J.row_ptr), dev(J.col_idx), dev(J.vals.reshape(-1)), dev(rhs)
x = torch.zeros(2 * J.n, dtype=torch.float64, device="cuda")
SETS = [dict(), dict(nu_pre=2, nu_post=2), dict(smoother=1), dict(smoother=1, cheb_degree=3),
        dict(theta=0.5), dict(interp_norm=0), dict(orth=1), dict(smoother=1, cheb_lo=0.1)]
if a.sets != "all":
    SETS = [SETS[int(i)] for i in a.sets.split(",")]
if a.opts:
    def _val(v):
        return float(v) if "." in v or "e" in v else int(v)
    SETS = [{k: _val(v) for k, v in (kv.split("=") for kv in grp.split(",") if kv)} for grp in a.opts.split(";")]
t_gen = time.perf_counter()
for opts in SETS:
    try:
        o = bf.bf_default_options(**opts)
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            h = bf.bf_setup(rp, ci, v, prob.dims, opt=o)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            x.zero_()
            r = bf.bf_solve(h, b, x, 1e-8, a.restart, a.maxit)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            bf.bf_destroy(h)
        print(f"C{a.config} m={a.restart} {str(opts):45s} iters {r['iters']:5d} conv {r['converged']} setup {1e3*(t1-t0):7.1f} ms "
              f"solve {1e3*(t2-t1):8.1f} ms  ms/iter {1e3*(t2-t1)/max(r['iters'],1):.3f}", flush=True)
    except Exception as e:
        print(f"C{a.config} {opts} failed: {e}", flush=True)
