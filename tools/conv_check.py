"""Residual history of the default solver on a config (prints every 100 iterations)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1611_00127_b200 as bf
from workload import make_system
cfg = int(sys.argv[1]); maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
dims = tuple(int(x) for x in sys.argv[3].split(",")) if len(sys.argv) > 3 else None
opts = dict(kv.split("=") for kv in sys.argv[4].split(",")) if len(sys.argv) > 4 else {}
opts = {k: (float(v) if "." in v else int(v)) for k, v in opts.items()}
prob, J, rhs = make_system(cfg, dims=dims)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
h = bf.bf_setup(dev(J.row_ptr), dev(J.col_idx), dev(J.vals.reshape(-1)), prob.dims, opt=bf.bf_default_options(**opts))
x = torch.zeros(2 * J.n, dtype=torch.float64, device="cuda")
t0 = time.perf_counter()
r = bf.bf_solve(h, dev(rhs), x, 1e-8, 30, maxit)
t1 = time.perf_counter()
hist = r["hist"]
print(f"C{cfg} {prob.dims} opts={opts} iters={r['iters']} conv={r['converged']} relres={r['relres']:.3e} solve {t1-t0:.2f}s")
print(" ".join(f"{k}:{hist[k]:.1e}" for k in range(0, len(hist), 100)))
