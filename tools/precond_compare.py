"""BF vs CPR-AMG(1) vs CPR-AMG(2) on the BJ configs: the comparison
pattern of the paper's Tables 3-5 (linear iterations per preconditioner) on the
synthetic stand-in fields, with B200 setup/solve times and the per-apply cost (CUDA events on
the solver stream).  One JSON line per (config, preconditioner).

    python tools/precond_compare.py --configs 1,2,3,4 [--maxit 1500]
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

NAMES = {0: "BF (Alg. 3)", 1: "CPR-AMG(1) (Alg. 1)", 2: "CPR-AMG(2) (Alg. 2)", 3: "coupled point AMG"}

p = argparse.ArgumentParser()
p.add_argument("--configs", type=str, default="1,2,3,4")
p.add_argument("--maxit", type=int, default=1500)
p.add_argument("--smoother", type=int, default=0)
p.add_argument("--preconds", type=str, default="0,1,2,3")
p.add_argument("--grids", type=str, default=None,
               help="mesh-independence study: ';'-separated grids for every config, e.g. '32,32,32;64,64,64'")
p.add_argument("--amg-maxit", type=int, default=300, help="cap for the coupled AMG (it stagnates)")
a = p.parse_args()
grids = [tuple(int(x) for x in g.split(",")) for g in a.grids.split(";")] if a.grids else [None]
for cfg, grid in ((int(c), g) for c in a.configs.split(",") for g in grids):
    prob, J, rhs = make_system(cfg, dims=grid)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    rp, ci, v, b = dev(J.row_ptr), dev(J.col_idx), dev(J.vals.reshape(-1)), dev(rhs)
    x = torch.zeros(2 * J.n, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    for pc in (int(q) for q in a.preconds.split(",")):
        maxit = a.amg_maxit if pc == 3 else a.maxit
        o = bf.bf_default_options(precond=pc, timing=1, smoother=a.smoother)
        for rep in range(2):  # second repetition reported (allocator and graph warm)
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            torch.cuda.synchronize()
            e[0].record(s)
            h = bf.bf_setup(rp, ci, v, prob.dims, opt=o)
            e[1].record(s)
            x.zero_()
            r = bf.bf_solve(h, b, x, 1e-8, 30, maxit)
            e[2].record(s)
            torch.cuda.synchronize()
            ams, na, aby = bf.bf_kernel_time(h, 2)
            lv = [bf.bf_num_levels(h, w) for w in range(4)]
            bf.bf_destroy(h)
        print(json.dumps({"config": cfg, "dims": prob.dims, "cells": J.n, "precond": NAMES[pc], "smoother": a.smoother,
                          "iters": r["iters"], "converged": r["converged"], "relres": r["relres"],
                          "setup_ms": e[0].elapsed_time(e[1]), "solve_ms": e[1].elapsed_time(e[2]),
                          "ms_per_iter": e[1].elapsed_time(e[2]) / max(r["iters"], 1),
                          "apply_us": 1e3 * ams / na if na else None,
                          "apply_model_gbs": (aby / na) / (ams / na / 1e3) / 1e9 if na and ams else None,
                          "levels": {"A_ss": lv[0], "S~": lv[1], "A_pp": lv[2], "J": lv[3]}}), flush=True)
