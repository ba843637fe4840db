"""Summarise an ncu --metrics gpu__time_duration.sum(,dram bytes) --csv launch list:
per-kernel count, total device ms, total DRAM GB (serialised, cold-cache: use shares)."""
import collections
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[i]
    ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[i + 1:]:
        per[int(r[idi])][r[mi]] = float(r[vi].replace(",", ""))
        names[int(r[idi])] = r[ki].split("(")[0][:70]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for k, m in per.items():
        a = agg[names[k]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0) / 1e6
        a[2] += (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e9
    tot = sum(a[1] for a in agg.values())
    print("%6s %10s %6s %9s  %s" % ("count", "ms", "share", "DRAM GB", "kernel"))
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print("%6d %10.3f %5.1f%% %9.3f  %s" % (a[0], a[1], 100 * a[1] / tot, a[2], n))
    print("total %.3f ms over %d launches" % (tot, len(per)))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
