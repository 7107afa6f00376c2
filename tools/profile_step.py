"""One BF-AMG-GMRES step (setup + `maxit` GMRES iterations) for ncu / nsys-less profiling.

    python tools/profile_step.py --config 3 --maxit 30 [--warm 1]

With --warm 1 a full untimed step runs first (ncu: skip its launches with -s)."""
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
p.add_argument("--maxit", type=int, default=30)
p.add_argument("--warm", type=int, default=0)
p.add_argument("--opts", type=str, default="")
a = p.parse_args()
dims = tuple(int(x) for x in a.dims.split(",")) if a.dims else None
prob, J, rhs = make_system(a.config, dims=dims)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
rp, ci, v, b = dev(J.row_ptr), dev(J.col_idx), dev(J.vals.reshape(-1)), dev(rhs)
x = torch.zeros(2 * J.n, dtype=torch.float64, device="cuda")
opts = dict(kv.split("=") for kv in a.opts.split(",") if kv)
opt = bf.bf_default_options(**{k: type(getattr(bf.bf_default_options(), k))(float(v)) if "." in v else int(v)
                               for k, v in opts.items()})
for w in range(a.warm + 1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = bf.bf_setup(rp, ci, v, prob.dims, opt=opt)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    x.zero_()
    r = bf.bf_solve(h, b, x, 1e-8, 30, a.maxit)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    nl = [bf.bf_num_levels(h, k) for k in (0, 1)]
    sizes = [[(bf.bf_get_level(h, k, l)["n"], len(bf.bf_get_level(h, k, l)["A"][1])) for l in range(nl[k])]
             for k in (0, 1)]
    print(f"run {w}: setup {1e3*(t1-t0):.1f} ms, solve {1e3*(t2-t1):.1f} ms, iters {r['iters']}, "
          f"relres {r['relres']:.3e}, launches {bf.bf_launch_count(h)}, levels {sizes}", flush=True)
    bf.bf_destroy(h)
