"""Tabulate key metrics of every kernel in an ncu --set full report."""
import csv
import subprocess
import sys

M = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "rdMB"), ("dram__bytes_write.sum", "wrMB"),
     ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
     ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1wf%"),
     ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
     ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "lsb"),
     ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "bar"),
     ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "ssb"),
     ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "mio"),
     ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
     ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid")]


def main(path, n=60):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    print("%-28s" % "kernel" + "".join("%9s" % lab for _, lab in M))
    for r in rows[2:2 + n]:
        vals = []
        for m, lab in M:
            try:
                v = float(r[h.index(m)].replace(",", ""))
            except (ValueError, IndexError):
                v = float("nan")
            vals.append(v)
        name = r[h.index("Kernel Name")]
        # keep the template arguments visible: k_csr_tma<3, 16, 2, 256>(...) -> k_csr_tma<3,16,2,256>
        name = name.replace("void ", "").replace("bf::", "").split("(")[0].replace(", ", ",")
        print("%-28s" % name[:28] + "".join("%9.1f" % v for v in vals))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 60)
