"""Per-config GPU-vs-oracle table (SURVEY 8(d) "Reporting"): for each BASELINE
configuration C1..C5 the GPU setup / solve time (CUDA events on the solver stream, median of
`--reps` after one warm-up), the GMRES(restart) iteration count to 1e-8, DOF-iterations/s, the J SpMV
rate (event-timed class 0), and -- for the configurations named in --oracle -- the CPU oracle
(plain C, 1 thread) run IN FULL on this box's host cores with parity of the two runs (iterations,
per-field solution difference).  One JSON line per configuration.

    python tools/config_table.py --configs 1,2,3,4,5 --oracle 1,2,4

C5 uses GMRES(200) (DESIGN 10.5: GMRES(30) stagnates at 1.3e-4 on J(u_0)); every other
configuration GMRES(30).  This tool is a measurement script (it may call the oracle: it is not
the product path).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1611_00127_b200 as bf
from workload import make_system

p = argparse.ArgumentParser()
p.add_argument("--configs", type=str, default="1,2,3,4,5")
p.add_argument("--oracle", type=str, default="1,2")
p.add_argument("--reps", type=int, default=3)
p.add_argument("--maxit", type=int, default=2500)
p.add_argument("--out", type=str, default=None)
a = p.parse_args()
want_oracle = {int(c) for c in a.oracle.split(",") if c}
out = open(a.out, "w") if a.out else None


def host_cpu():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return f"{model}, nproc {os.cpu_count()}"


for cfg in (int(c) for c in a.configs.split(",")):
    prob, J, rhs = make_system(cfg)
    restart = 200 if cfg == 5 else 30
    N = 2 * J.n
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    rp, ci, v, b = dev(J.row_ptr), dev(J.col_idx), dev(J.vals.reshape(-1)), dev(rhs)
    x = torch.zeros(N, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    o = bf.bf_default_options(timing=1)
    su, so, its = [], [], []
    reps = 1 if cfg == 5 else a.reps
    for rep in range(reps + 1):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        torch.cuda.synchronize()
        e[0].record(s)
        h = bf.bf_setup(rp, ci, v, prob.dims, opt=o)
        e[1].record(s)
        x.zero_()
        r = bf.bf_solve(h, b, x, 1e-8, restart, a.maxit)
        e[2].record(s)
        torch.cuda.synchronize()
        if rep > 0 or reps == 1:
            su.append(e[0].elapsed_time(e[1]))
            so.append(e[1].elapsed_time(e[2]))
            its.append(r["iters"])
        k_ms, k_n, k_by = bf.bf_kernel_time(h, 0)     # J SpMV class: ms, launches, algorithmic bytes
        a_ms, a_n, a_by = bf.bf_kernel_time(h, 2)     # BF apply
        stats = [bf.bf_hierarchy_stats(h, w) for w in (0, 1)]
        bf.bf_destroy(h)
        if cfg == 5 and rep == 0:
            break
    xg = x.cpu().numpy()
    rec = {"config": f"C{cfg}", "dims": list(prob.dims), "dof": N, "restart": restart,
           "gpu_setup_ms": float(np.median(su)), "gpu_solve_ms": float(np.median(so)), "iters": int(np.median(its)),
           "converged": bool(r["converged"]), "relres": r["relres"],
           "dof_iters_per_s": N * float(np.median(its)) / (1e-3 * (np.median(su) + np.median(so))),
           "spmv_us": 1e3 * k_ms / k_n if k_n else None,
           "spmv_model_gbs": (k_by / k_n) / (k_ms / k_n * 1e-3) / 1e9 if k_n and k_ms else None,
           "apply_us": 1e3 * a_ms / a_n if a_n else None,
           "apply_model_gbs": (a_by / a_n) / (a_ms / a_n * 1e-3) / 1e9 if a_n and a_ms else None,
           "operator_complexity": [st.get("operator_complexity") for st in stats] if isinstance(stats[0], dict) else None}
    if cfg in want_oracle:
        import oracle
        t0 = time.perf_counter()
        ob = oracle.BF(J)
        t1 = time.perf_counter()
        ro = ob.gmres(rhs, tol=1e-8, restart=restart, maxit=a.maxit)
        t2 = time.perf_counter()
        xo = ro["x"]
        rec.update({"oracle_setup_s": t1 - t0, "oracle_solve_s": t2 - t1, "oracle_iters": ro["iters"],
                    "oracle_converged": bool(ro["converged"]), "oracle_cores": 1, "oracle_host": host_cpu(),
                    "oracle_dof_iters_per_s": N * ro["iters"] / (t2 - t0),
                    "parity": {"iters_diff": int(r["iters"] - ro["iters"]),
                               "x_rel_diff_p": float(np.linalg.norm(xg[0::2] - xo[0::2]) / np.linalg.norm(xo[0::2])),
                               "x_rel_diff_s": float(np.linalg.norm(xg[1::2] - xo[1::2]) / np.linalg.norm(xo[1::2]))}})
        del ob
    line = json.dumps(rec)
    print(line, flush=True)
    if out:
        out.write(line + "\n")
        out.flush()
    del rp, ci, v, b, x
    torch.cuda.empty_cache()
