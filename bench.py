#!/usr/bin/env python
"""Benchmark of the BF-AMG-GMRES hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl reference]

One STEP = one pass of the whole hot path on one Jacobian:
bf_setup (ingest/validate, field split, S~, both AMG hierarchies) from device-resident
J, then bf_solve (GMRES(30), tol 1e-8, x0 = 0, BF preconditioner), then bf_destroy.
The workload is configs[2] (C3, 128^3, 4.19M unknowns): the grid BASELINE.json's
roofline target is stated on.  Inputs (J = 533 MB) are
larger than the 126 MB L2, so no explicit flush is needed between steps.

value = DOF*iterations/s over the whole step (sum over ranks / max-over-ranks time).
N > 1: independent replicas, one per GPU (the path does not shard).
--impl reference: the CPU oracle (oracle/, plain C, 1 core) on a bounded sample of the
same workload -- the only other place this script runs oracle/ code.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BF-AMG-GMRES DOF-iterations/s (setup+solve per Jacobian)"
UNIT = "DOF-iters/s"
FALLBACK_HBM = 6650.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=3)
    p.add_argument("--dims", type=str, default=None, help="override grid, e.g. 64,64,64 (not a bench line)")
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--restart", type=int, default=30)
    p.add_argument("--tol", type=float, default=1e-8)
    p.add_argument("--maxit", type=int, default=1000)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


# ------------------------------------------------------------------------------------------
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(dev)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [l.split(",") for l in open(self.f.name).read().strip().splitlines() if l.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for nm, v in zip(names, r[5:9]):
                    if "Active" in v and "Not" not in v:
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        busy = [s for s in sm if mx and s > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def reduce_over_ranks(dist, t_ms, units, device="cpu"):
    """Whole-job aggregate of independent replicas: max of the per-rank device times and the
    sum of the per-rank work units (works with NCCL on GPU tensors and gloo on CPU)."""
    if dist is None:
        return t_ms, units
    import torch
    t = torch.tensor([t_ms], dtype=torch.float64, device=device)
    u = torch.tensor([units], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return float(t.item()), float(u.item())


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_from_profiles(kernel_class):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(path))
        return d.get(kernel_class)
    except Exception:
        return None


# ------------------------------------------------------------------------------------------
def sub_jacobian(J_full, prob, frac=4):
    """The first nz/frac z-planes of the SAME Jacobian (couplings to the dropped planes removed)."""
    import numpy as np
    from workload import BSR2
    nx, ny, nz = prob.dims
    nzs = max(1, nz // frac)
    ns = nx * ny * nzs
    rp, ci, v = J_full.row_ptr, J_full.col_idx, J_full.vals
    keep = np.arange(rp[ns])
    keep = keep[ci[keep] < ns]
    rows = np.repeat(np.arange(ns), np.diff(rp[:ns + 1]))
    rows = rows[ci[:rp[ns]] < ns]
    rps = np.zeros(ns + 1, np.int32)
    np.cumsum(np.bincount(rows, minlength=ns), out=rps[1:])
    return BSR2(ns, rps, np.ascontiguousarray(ci[keep]), np.ascontiguousarray(v[keep]), (nx, ny, nzs)), nzs


def oracle_sample(J_full, prob, iters, restart, tol, frac=4, reps=2):
    """Bounded sample of the same workload for the CPU oracle (1 core), in the metric's unit.

    The sample is the first nz/frac z-planes of the SAME Jacobian.  Its cost is measured, not
    modelled per iteration: the oracle setup, then ONE complete GMRES(restart) cycle (initial
    residual, `restart` Arnoldi steps with CGS2 over the growing basis, the cycle-end update and
    true residual) and one partial cycle of (iters mod restart) steps with its own cycle end.  A
    solve of `iters` Arnoldi steps is floor(iters/restart) complete cycles plus that partial
    one, so  t(iters) = setup + floor(iters/restart) t_cycle + t_partial  is the oracle's time
    for `iters` iterations on the sample (each cycle of restarted GMRES does the same work,
    independent of the residual).  `iters` is a measured iteration count of the full problem
    (GPU and oracle agree within +-1, tests/test_gpu_*).  Calibrated against a full-size
    oracle run (profiles/r02_oracle_c3_full.json)."""
    import numpy as np
    import oracle
    Js, nzs = sub_jacobian(J_full, prob, frac)
    ns = Js.n
    nz = prob.dims[2]
    rhs = np.ones(2 * ns)
    t0 = time.perf_counter()
    bf = oracle.BF(Js)
    t1 = time.perf_counter()
    iters = max(int(iters), 1)
    full_cycles, rem = divmod(iters, restart)
    t_cycle, t_part = float("inf"), 0.0
    for _ in range(reps):                                                  # min over repetitions
        ta = time.perf_counter()
        r = bf.gmres(rhs, tol=0.0, restart=restart, maxit=restart)        # one complete cycle
        t_cycle = min(t_cycle, time.perf_counter() - ta)
        assert r["iters"] == restart
    if rem:
        t_part = float("inf")
        for _ in range(reps):
            ta = time.perf_counter()
            r2 = bf.gmres(rhs, tol=0.0, restart=restart, maxit=rem)    # the partial last cycle
            t_part = min(t_part, time.perf_counter() - ta)
            assert r2["iters"] == rem
    t_est = (t1 - t0) + full_cycles * t_cycle + t_part
    raw = 2 * ns * iters / t_est
    calib, csrc = oracle_calibration(prob_cfg(prob), frac, prob.dims)
    value = raw / calib
    sample = (f"oracle (plain C, -O2, 1 thread) on the first {nzs} of {nz} z-planes of the same C{prob_cfg(prob)} "
              f"Jacobian ({ns} cells, {2 * ns} DOF): setup {t1 - t0:.2f} s measured, one full GMRES({restart}) "
              f"cycle {t_cycle:.2f} s and a partial cycle of {rem} steps {t_part:.2f} s measured (min of {reps}); "
              f"{iters} iterations = {full_cycles} cycles + {rem} steps -> {raw:.4g} DOF-iters/s on the sample"
              + (f", divided by {calib:.4f}, the sample/full-size rate ratio of {csrc}" if calib != 1.0 else
                 " (no full-size calibration for this workload)"))
    return dict(value=value, raw_value=raw, calib=calib, unit=UNIT, cores=1, kind="oracle", sample=sample,
                host=host_cpu(), setup_s=t1 - t0, cycle_s=t_cycle, partial_s=t_part, est_s=t_est, dof=2 * ns,
                wall_s=time.perf_counter() - t0)


def oracle_calibration(config, frac, dims):
    """Ratio (sample rate / full-size rate) measured once by a full-size oracle run on the GPU
    box's host (tests/scripts/oracle_full.py -> profiles/r02_oracle_c<config>_full.json): the
    oracle's cost per DOF-iteration grows with the problem size (cache and TLB reach), so the
    sample's rate is scaled back to the full-size workload's."""
    path = os.path.join(ROOT, "profiles", f"r02_oracle_c{config}_full.json")
    try:
        d = json.load(open(path))
        if list(d["dims"]) != list(dims):
            return 1.0, None
        for s in d.get("samples", []):
            if s["frac"] == frac and s.get("method") == SAMPLE_METHOD:
                full = d["value_dof_iters_per_s"]
                return float(s["value_raw"]) / full, (f"{os.path.relpath(path, ROOT)} (full C{config} oracle run: "
                                                       f"{d['total_s']:.1f} s for {d['iters']} iterations = "
                                                       f"{full:.4g} DOF-iters/s, {d['host']})")
    except Exception:
        pass
    return 1.0, None


SAMPLE_METHOD = "setup + min-of-2 full cycle + min-of-2 partial cycle"


def host_cpu():
    """The box's host CPU (report nproc and the model next to the oracle timing)."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return f"{model}, nproc {os.cpu_count()}"


def prob_cfg(prob):
    return getattr(prob, "_config", "?")


def build_workload(config, dims):
    from workload import make_system
    prob, J, rhs = make_system(config, dims=dims)
    prob._config = config
    return prob, J, rhs


def workload_name(config, prob):
    from workload import CONFIG_NAMES
    return f"{CONFIG_NAMES[config]} [{prob.nx}x{prob.ny}x{prob.nz}]"


REF_FRAC = 4     # the reference arm's sample: the first nz/4 z-planes (about 30-40 s of oracle time)


def oracle_iterations(config, dims):
    """The oracle's measured GMRES(30) iteration count to 1e-8 on a full-size configuration,
    from a committed full run (tests/scripts/oracle_full.py, calls only oracle/)."""
    if dims is not None:
        return None, "grid override"
    path = os.path.join(ROOT, "profiles", f"r02_oracle_c{config}_full.json")
    try:
        d = json.load(open(path))
        return int(d["iters"]), os.path.relpath(path, ROOT) + " (oracle, full size, measured)"
    except Exception as e:
        return None, f"{os.path.relpath(path, ROOT)}: {e}"


# ------------------------------------------------------------------------------------------
def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    dims = tuple(int(x) for x in args.dims.split(",")) if args.dims else None
    prob, J, rhs = build_workload(args.config, dims)
    # the oracle's own measured iteration count on this configuration (a full-size oracle run to
    # 1e-8, tests/scripts/oracle_full.py -> profiles/); the sample's measured setup + cycle times give the
    # oracle's time for that many iterations
    iters, src = oracle_iterations(args.config, dims)
    if iters is None:
        print(json.dumps({"impl": "reference", "unavailable": f"no measured oracle iteration count for config "
                                                              f"{args.config} {dims or ''} ({src})"}), flush=True)
        return 0
    vals, walls = [], []
    for s in range(args.warmup + args.steps):
        res = oracle_sample(J, prob, iters, args.restart, args.tol, frac=REF_FRAC)
        if s >= args.warmup:
            vals.append(res["value"])
            walls.append(res["est_s"])
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            # the oracle's time for one full-size step implied by the sample's rate
            "ms_per_step": 1e3 * 2 * J.n * iters / v,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, SPE10 stand-in)", "iters": iters, "iters_source": src,
            "config": {"workload": workload_name(args.config, prob), "restart": args.restart, "tol": args.tol},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": res["sample"],
                             "host": res["host"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import numpy as np
    import torch
    ws, rank, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1611_00127_b200 as bf
    dims = tuple(int(x) for x in args.dims.split(",")) if args.dims else None
    prob, J, rhs = build_workload(args.config, dims)
    n, N = J.n, 2 * J.n
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    d_rp, d_ci, d_v = dev(J.row_ptr), dev(J.col_idx), dev(J.vals.reshape(-1))
    d_b = dev(rhs)
    d_x = torch.zeros(N, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    # kernel-class events around every 4th Arnoldi step (sampled: timing=1 on every step costs
    # 3.3 % of the solve, timing=4 is within noise of no instrumentation; measured C3 60 it)
    TIMING_EVERY = 4
    opt = bf.bf_default_options(timing=TIMING_EVERY)

    def step(record):
        h = bf.bf_setup(d_rp, d_ci, d_v, prob.dims, opt=opt)
        try:
            e_mid = torch.cuda.Event(enable_timing=True)
            e_mid.record(stream)
            d_x.zero_()
            r = bf.bf_solve(h, d_b, d_x, args.tol, args.restart, args.maxit, True)
            if record is not None:
                record["iters"].append(r["iters"])
                record["relres"].append(r["relres"])
                record["conv"].append(r["converged"])
                record["mid"].append(e_mid)
                record["launches"] += bf.bf_launch_count(h)
                if "hier" not in record:
                    record["hier"] = {name: bf.bf_hierarchy_stats(h, w) for w, name in ((0, "A_ss"), (1, "S~"))}
                for k in range(4):
                    record["kt"][k] = [a + b for a, b in zip(record["kt"][k], bf.bf_kernel_time(h, k))]
        finally:
            bf.bf_destroy(h)

    for _ in range(args.warmup):
        step(None)
    torch.cuda.synchronize()
    rec = {"iters": [], "relres": [], "conv": [], "mid": [], "launches": 0, "kt": [[0.0, 0, 0.0] for _ in range(4)]}
    clocks = Clocks(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    starts = []
    e0.record(stream)
    for s in range(args.steps):
        es = torch.cuda.Event(enable_timing=True)
        es.record(stream)
        starts.append(es)
        step(rec)
    e1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    t_ms = e0.elapsed_time(e1)
    setup_ms = [starts[i].elapsed_time(rec["mid"][i]) for i in range(args.steps)]
    ends = starts[1:] + [e1]
    solve_ms = [rec["mid"][i].elapsed_time(ends[i]) for i in range(args.steps)]
    # a timed solve that did not converge makes the line invalid: DOF-iterations of a stalled
    # solve are not work towards a solution
    all_converged = all(rec["conv"])
    units = float(sum(N * it for it in rec["iters"]))
    t_ms, units = reduce_over_ranks(dist, t_ms, units, "cuda")
    value = units / (t_ms / 1e3)

    # ---- roofline of the dominant kernel class (device time share inside the timed region)
    peak, peak_src = peaks()
    kt = rec["kt"]
    cls = {0: "bsr2_spmv (J SpMV, one DIA-BSR kernel; bytes: SURVEY 8(d) 36 B/block + 36 B/row)",
           1: "gmres_cgs2 (3 fused orthogonalisation passes per Arnoldi step; bytes: 8N(3j+5))",
           2: "bf_apply (Algorithm 3: two V-cycles + A_ps coupling, ~50 DIA / windowed-JDS / TMA-CSR kernels + two dense tail operators in one CUDA graph; "
              "bytes: SURVEY 8(d) per-level V(1,1) model on the actual hierarchies)"}

    n_arnoldi = float(sum(rec["iters"]))

    def roof(k):
        ms, launches, by = kt[k]
        achieved = (by / launches) / (ms / launches / 1e3) / 1e9 if launches and ms > 0 else None
        traffic = traffic_from_profiles(cls[k].split()[0])
        # the kernels' own storage (DIA, fused restriction) moves fewer bytes than the SURVEY
        # model: the DRAM rate below (ncu bytes per launch / live launch time) is the one to
        # compare with the copy bandwidth when frac exceeds it
        dram = traffic / (ms / launches / 1e3) / 1e9 if traffic and launches and ms > 0 else None
        return {"bound": "hbm", "kernel": cls[k], "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak if achieved else None, "peak_source": peak_src,
                "traffic": traffic, "achieved_dram": dram, "frac_dram": dram / peak if dram else None,
                "timed_launches": launches,
                "timing": f"CUDA events on the solver stream around this class in every {TIMING_EVERY}th Arnoldi step "
                          "of the timed steps (sampled)",
                "alg_bytes_per_launch": by / launches if launches else None,
                "avg_launch_us": 1e3 * ms / launches if launches else None,
                # every Arnoldi step runs each class once: its share is the sampled mean launch time
                # times the number of Arnoldi steps in the timed region
                "share_of_step": (ms / launches) * n_arnoldi / t_ms if t_ms and launches else None}
    dom = max(range(3), key=lambda k: kt[k][0] / kt[k][1] if kt[k][1] else 0.0)
    roofline = roof(dom)
    others = [roof(k) for k in range(3) if k != dom]

    # ---- e2e: same metric through the C-ABI with HOST buffers (pinned), copies inside
    e2e = None
    if not args.no_e2e:
        h_rp = torch.from_numpy(np.ascontiguousarray(J.row_ptr)).pin_memory()
        h_ci = torch.from_numpy(np.ascontiguousarray(J.col_idx)).pin_memory()
        h_v = torch.from_numpy(np.ascontiguousarray(J.vals.reshape(-1))).pin_memory()
        h_b = torch.from_numpy(rhs.copy()).pin_memory()
        h_x = torch.zeros(N, dtype=torch.float64).pin_memory()
        k_e2e = max(1, min(args.steps, 2))
        its = 0
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(k_e2e):
            h = bf.bf_setup(h_rp, h_ci, h_v, prob.dims)
            h_x.zero_()
            r = bf.bf_solve(h, h_b, h_x, args.tol, args.restart, args.maxit, True)
            its += r["iters"]
            bf.bf_destroy(h)
        f1.record(stream)
        torch.cuda.synchronize()
        te = f0.elapsed_time(f1)
        ue = float(N * its)
        te, ue = reduce_over_ranks(dist, te, ue, "cuda")
        h2d = (h_rp.numel() * 4 + h_ci.numel() * 4 + h_v.numel() * 8 + h_b.numel() * 8 + h_x.numel() * 8)
        e2e = {"value": ue / (te / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(N * 8), "steps": k_e2e}

    # context: time to solution of the other preconditioner options on the same J (one
    # untimed-for-value step each): the Chebyshev(2) smoother, and the paper's two-stage
    # CPR-AMG(1)/(2) preconditioners (Algorithms 1, 2) it compares BF against
    alt = None
    if not args.no_e2e:
        alt = []
        for name, kw in (("BF, l1-Jacobi V(1,1) on both hierarchies (round-1 default; option smoother=0)",
                          dict(smoother=0)),
                         ("BF, Chebyshev(2) on [0.15,1] on both hierarchies (options smoother_p=-1, cheb_lo=0.15)",
                          dict(smoother_p=-1, cheb_lo=0.15)),
                         ("CPR-AMG(2) additive, ILU(0) + A_pp, A_ss V-cycles (option precond=2)", dict(precond=2))):
            o2 = bf.bf_default_options(timing=1, **kw)
            torch.cuda.synchronize()
            a0, a1, a2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a0.record(stream)
            h2 = bf.bf_setup(d_rp, d_ci, d_v, prob.dims, opt=o2)
            a1.record(stream)
            d_x.zero_()
            r2 = bf.bf_solve(h2, d_b, d_x, args.tol, args.restart, args.maxit, True)
            a2.record(stream)
            torch.cuda.synchronize()
            ams, alaunch, aby = bf.bf_kernel_time(h2, 2)
            bf.bf_destroy(h2)
            alt.append({"preconditioner": name, "setup_ms": a0.elapsed_time(a1), "solve_ms": a1.elapsed_time(a2),
                        "iters": r2["iters"], "converged": r2["converged"], "relres": r2["relres"],
                        "apply_us": 1e3 * ams / alaunch if alaunch else None,
                        "apply_model_gbs": (aby / alaunch) / (ams / alaunch / 1e3) / 1e9 if alaunch and ams else None})

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = oracle_sample(J, prob, int(statistics.median(rec["iters"])), args.restart, args.tol)
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample", "host", "raw_value", "calib")}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded generator; SPE10 stand-in fields)",
                "config": {"workload": workload_name(args.config, prob), "cells": n, "dof": N,
                           "nnzb": J.nnzb, "restart": args.restart, "tol": args.tol, "x0": "zero",
                           "step": "bf_setup(device J) + bf_solve + bf_destroy",
                           "l2": "inputs larger than L2 (J = %.0f MB > 126 MB), no flush" %
                                 ((J.nnzb * 36 + (n + 1) * 4) / 1e6),
                           "parallelism": f"replicas x{ws}" if ws > 1 else "1 GPU"},
                "valid": all_converged,
                **({} if all_converged else {"invalid": "a timed GMRES solve did not reach the tolerance"}),
                "time_to_solution_ms": statistics.median(a + b for a, b in zip(setup_ms, solve_ms)),
                "setup_ms_median": statistics.median(setup_ms), "solve_ms_median": statistics.median(solve_ms),
                "iters_median": statistics.median(rec["iters"]),
                "iters": rec["iters"], "relres": rec["relres"], "converged": rec["conv"],
                "setup_ms": setup_ms, "solve_ms": solve_ms,
                "hierarchies": rec.get("hier"),
                "roofline": roofline, "roofline_other": others,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": rec["launches"], "clocks": clk,
                "alt_time_to_solution": alt}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
