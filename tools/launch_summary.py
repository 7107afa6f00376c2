"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name."""
import collections
import csv
import sys


def summarise(path, top=45, title=""):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    H = rows[hdr]
    ki, mi, ui = H.index("Kernel Name"), H.index("Metric Value"), H.index("Metric Unit")
    mn = H.index("Metric Name") if "Metric Name" in H else None
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[hdr + 1:]:
        if len(r) <= mi or (mn is not None and r[mn] != "gpu__time_duration.sum"):
            continue
        v = float(r[mi].replace(",", ""))
        u = r[ui]
        v = v / 1e3 if u in ("nsecond", "ns") else (v * 1e3 if u in ("msecond", "ms") else v)
        name = r[ki].split("(")[0][:80]
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    out = [f"# {title}", f"# total {tot:.0f} us over {sum(a[0] for a in agg.values())} launches (units: us)"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{t:10.1f} us {100 * t / tot:5.1f}%  n={n:5d}  avg={t / n:9.2f} us  {k}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1], title=" ".join(sys.argv[2:])))
