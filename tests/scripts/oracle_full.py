"""Full-size oracle run to convergence (test infrastructure: calls only oracle/ and workload/).

    python tests/scripts/oracle_full.py --config 3 [--out profiles/r02_oracle_c3_full.json]

Times the CPU oracle (plain C, 1 thread) on the whole BASELINE.json configuration: bf_setup
equivalent (split, S~, both AMG hierarchies) and GMRES(30) to 1e-8 from x0 = 0, and records the
measured iteration count.  Then times bench.py's bounded sample (first nz/frac z-planes, one
complete GMRES cycle + the partial cycle) with that iteration count, so the sample's
extrapolation can be checked against the measured full run (within 5 %).
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
import bench  # noqa: E402
from workload import make_system  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=3)
p.add_argument("--maxit", type=int, default=2000)
p.add_argument("--out", type=str, default=None)
p.add_argument("--fracs", type=str, default="4,8")
a = p.parse_args()

t_gen = time.perf_counter()
prob, J, rhs = make_system(a.config)
prob._config = a.config
t_gen = time.perf_counter() - t_gen
t0 = time.perf_counter()
bf = oracle.BF(J)
t1 = time.perf_counter()
r = bf.gmres(rhs, tol=1e-8, restart=30, maxit=a.maxit)
t2 = time.perf_counter()
true_rel = float(np.linalg.norm(rhs - bf.spmv(r["x"])) / np.linalg.norm(rhs))
N = 2 * J.n
rec = {"config": a.config, "dims": list(prob.dims), "dof": N, "impl": "oracle (plain C, gcc -O2 -ffp-contract=off, 1 thread)",
       "host": bench.host_cpu(), "setup_s": t1 - t0, "solve_s": t2 - t1, "total_s": t2 - t0,
       "iters": r["iters"], "converged": r["converged"], "relres": r["relres"], "true_relres": true_rel,
       "value_dof_iters_per_s": N * r["iters"] / (t2 - t0), "levels": [bf.nlev(0), bf.nlev(1)],
       "hist_every_30": [float(h) for h in r["hist"][::30]], "generator_s": t_gen, "samples": []}
print(json.dumps({k: v for k, v in rec.items() if k != "hist_every_30"}), flush=True)
for frac in (int(f) for f in a.fracs.split(",")):
    s = bench.oracle_sample(J, prob, r["iters"], 30, 1e-8, frac=frac)
    rec["samples"].append({"frac": frac, "value_raw": s["raw_value"], "method": bench.SAMPLE_METHOD,
                           "ratio_to_full": s["raw_value"] / rec["value_dof_iters_per_s"],
                           "sample": s["sample"], "wall_s": s["wall_s"], "setup_s": s["setup_s"],
                           "cycle_s": s["cycle_s"], "partial_s": s["partial_s"]})
    print(json.dumps(rec["samples"][-1]), flush=True)
if a.out:
    with open(a.out, "w") as f:
        json.dump(rec, f, indent=1)
