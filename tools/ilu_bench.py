"""Time the CPR block-ILU(0) sweeps (bf_ilu_solve: forward + backward + copy-out) on one config.
Sweep knobs are environment variables read once per process: BF_ILU_CTAS, BF_ILU_SLEEP,
BF_ILU_FLAGS.  J is cached in /tmp between processes.

    python tools/ilu_bench.py --config 3 [--reps 20]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1611_00127_b200 as bf
from workload import make_system, seeded_vector

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=3)
p.add_argument("--reps", type=int, default=20)
a = p.parse_args()
cache = f"/tmp/bf_J_c{a.config}.npz"
if os.path.exists(cache):
    z = np.load(cache)
    rp, ci, vals, dims = z["rp"], z["ci"], z["vals"], tuple(z["dims"])
else:
    prob, J, rhs = make_system(a.config)
    rp, ci, vals, dims = J.row_ptr, J.col_idx, J.vals.reshape(-1), prob.dims
    np.savez(cache, rp=rp, ci=ci, vals=vals, dims=np.array(dims))
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
s = bf.BFSolver(dev(rp), dev(ci), dev(vals), dims, precond=1)
N = 2 * (len(rp) - 1)
r = dev(seeded_vector(N, 1))
x = torch.empty(N, dtype=torch.float64, device="cuda")
for _ in range(3):
    s.ilu_solve(r, x)
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(st)
for _ in range(a.reps):
    s.ilu_solve(r, x)
e1.record(st)
torch.cuda.synchronize()
print(json.dumps({"config": a.config, "ctas": os.environ.get("BF_ILU_CTAS", "4"), "sleep": os.environ.get("BF_ILU_SLEEP", "0"),
                  "flags": os.environ.get("BF_ILU_FLAGS", "0"), "ilu_solve_us": 1e3 * e0.elapsed_time(e1) / a.reps,
                  "levels": s.ilu(len(ci))[2]}), flush=True)
