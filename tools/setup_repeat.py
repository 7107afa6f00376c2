"""Repeated bf_setup/bf_destroy on one config (BF_VERBOSE=1 prints per-phase times)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1611_00127_b200 as bf
from workload import make_system
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
solve = len(sys.argv) > 2 and sys.argv[2] == "solve"
prob, J, rhs = make_system(cfg)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
rp, ci, v, b = dev(J.row_ptr), dev(J.col_idx), dev(J.vals.reshape(-1)), dev(rhs)
x = torch.zeros(2 * J.n, dtype=torch.float64, device="cuda")
for rep in range(int(os.environ.get("REPS", "6"))):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = bf.bf_setup(rp, ci, v, prob.dims)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    if solve:
        bf.bf_solve(h, b, x, 1e-8, 30, 60)
    print(f"rep {rep}: setup {1e3*(t1-t0):.1f} ms, device bytes {bf.bf_device_bytes(h)/1e9:.2f} GB", file=sys.stderr, flush=True)
    bf.bf_destroy(h)
