"""Summarise ncu --set full reports (one kernel each) into a text table:
duration, DRAM bytes, throughputs, hit rates, occupancy, top stall reasons.
python tools/ncu_summary.py OUT.txt REPORT.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("launches in report", "launches in report (longest shown)"),
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1TEX % peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "LTS % peak"),
    ("l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed", "L1->XBAR req % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads / instruction"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    # several launches in one report: the longest one
    k = hdr.index("gpu__time_duration.sum")
    vals = max(rows[2:], key=lambda r: float(r[k].replace(",", "") or 0))
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    d["launches in report"] = (str(len(rows) - 2), "")
    return d


def stalls(d):
    pre = "smsp__pcsamp_warps_issue_stalled_"
    items = [(k[len(pre):], float(v[0].replace(",", ""))) for k, v in d.items()
             if k.startswith(pre) and not k.endswith("_not_issued") and v[0]]
    tot = sum(x for _, x in items) or 1.0
    items.sort(key=lambda t: -t[1])
    return ", ".join("%s %.0f%%" % (n, 100 * x / tot) for n, x in items[:5])


def main():
    out = open(sys.argv[1], "w")
    for rep in sys.argv[2:]:
        d = raw(rep)
        out.write("## %s\n  kernel: %s\n" % (rep.split("/")[-1], d.get("Kernel Name", ("?",))[0]))
        for k, name in KEYS:
            if k in d:
                out.write("  %-24s %s %s\n" % (name, d[k][0], d[k][1]))
        out.write("  stalls (pc sampling): %s\n\n" % stalls(d))
    out.close()


if __name__ == "__main__":
    main()
