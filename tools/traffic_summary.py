"""DRAM bytes per launch of the three bench kernel classes, from an ncu launch list.

Input: the csv written by
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
      python tools/profile_step.py --config 3 --maxit 30
(setup, then one GMRES(30) cycle).  Classes (the same split bench.py's bf_kernel_time uses):
  bsr2_spmv  : the J SpMV kernels (k_bsr2_*), bytes per launch
  gmres_cgs2 : k_dots / k_axpy_dots / k_axpy_norm / k_scale / k_lincomb, bytes per Arnoldi step
  bf_apply   : every other kernel launched after the first J SpMV (split, V-cycle kernels, merge),
               bytes per apply (= per k_split_vec launch)
Usage: python tools/traffic_summary.py launches.csv > profiles/traffic.json
"""
import collections
import csv
import json
import sys

SPMV = ("k_bsr2_spmv", "k_bsr2_dia")
GMRES = ("k_dots", "k_axpy_dots", "k_axpy_norm", "k_scale", "k_lincomb")


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    H = rows[hdr]
    ii, ki, mn, mi, ui = (H.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    per = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= mi:
            continue
        nm = r[ki].split("(")[0].split("<")[0].strip()
        nm = nm.replace("void ", "").split("::")[-1]
        d = per.setdefault(r[ii], {"name": nm})
        v = float(r[mi].replace(",", ""))
        u = r[ui].lower()
        scale = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)
        d[r[mn]] = v * scale
    return list(per.values())


def summarise(path):
    ls = load(path)
    # the last step's solve only (with --warm k the list holds k+1 setups + solves): from the first J
    # SpMV after the last setup kernel
    last_setup = max((i for i, d in enumerate(ls) if d["name"].startswith(("k_pmis", "k_spgemm", "k_interp"))),
                     default=-1)
    first = next(i for i, d in enumerate(ls) if i > last_setup and d["name"] in SPMV)
    by = collections.defaultdict(float)
    cnt = collections.Counter()
    for d in ls[first:]:
        b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        n = d["name"]
        cls = "bsr2_spmv" if n in SPMV else "gmres_cgs2" if n.startswith(GMRES) else "bf_apply"
        by[cls] += b
        if n in SPMV:
            cnt["bsr2_spmv"] += 1
        if n.startswith("k_split_vec"):
            cnt["bf_apply"] += 1
        if n.startswith("k_axpy_norm"):
            cnt["gmres_cgs2"] += 1
    out = {k: by[k] / max(cnt[k], 1) for k in ("bsr2_spmv", "gmres_cgs2", "bf_apply")}
    out["_source"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (launch list of "
                      "tools/profile_step.py --config 3 --maxit 30); bytes per launch via tools/traffic_summary.py "
                      "(bf_apply: sum over its kernels per apply; gmres_cgs2: per Arnoldi step)")
    out["_counts"] = dict(cnt)
    return out


if __name__ == "__main__":
    print(json.dumps(summarise(sys.argv[1]), indent=1))
