"""Per-launch table from an `ncu --metrics ... --csv` log: time, DRAM bytes,
L2/L1 sector hit rates and threads per instruction (warp efficiency)."""
import collections
import csv
import sys

COLS = [("gpu__time_duration.sum", "ms", 1e-6), ("dram__bytes_read.sum", "dram_rd_GB", 1e-9),
        ("dram__bytes_write.sum", "dram_wr_GB", 1e-9), ("lts__t_sector_hit_rate.pct", "L2_hit_%", 1),
        ("l1tex__t_sector_hit_rate.pct", "L1_hit_%", 1),
        ("smsp__thread_inst_executed_per_inst_executed.ratio", "thr/inst", 1)]


def main(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[i]
    ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[i + 1:]:
        per[int(r[idi])][r[mi]] = float(r[vi].replace(",", ""))
        names[int(r[idi])] = r[ki].split("(")[0][:60]
    print("%4s %-60s " % ("id", "kernel") + " ".join("%10s" % c[1] for c in COLS))
    for k in sorted(per):
        m = per[k]
        print("%4d %-60s " % (k, names[k]) + " ".join(
            "%10.3f" % (m[c[0]] * c[2]) if c[0] in m else "%10s" % "-" for c in COLS))


if __name__ == "__main__":
    main(sys.argv[1])
