"""Summarise an ncu capture for profiles/: python profiles/summarize.py REP.ncu-rep LAUNCHES.csv OUT.md

Reads (here, no GPU needed) the `ncu --set full` report and the
`--metrics gpu__time_duration.sum` launch list that gpurun brought back, and
writes the per-kernel table the DESIGN/roofline numbers cite."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.per_cycle_active", "warps/SM"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads/inst"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp insts"),
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main(rep, launches, out):
    h, units, rows = raw_rows(rep)
    lines = ["| kernel | " + " | ".join(n for _, n in KEYS) + " | top stall reasons |",
             "|---" * (len(KEYS) + 2) + "|"]
    for r in rows:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        vals = []
        for k, _ in KEYS:
            v = r[h.index(k)] if k in h else ""
            u = units[h.index(k)] if k in h else ""
            vals.append(f"{v} {u}".strip())
        st = [(h[i].replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i])) for i in range(len(h))
              if "pcsamp_warps_issue_stalled" in h[i] and "not_issued" not in h[i] and r[i].replace(".", "").isdigit()]
        tot = sum(v for _, v in st) or 1
        top = ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in sorted(st, key=lambda x: -x[1])[:3])
        lines.append(f"| {name} | " + " | ".join(vals) + f" | {top} |")
    if launches == "-":  # no launch list for this capture
        open(out, "w").write("\n".join(lines) + "\n")
        return
    # launch list: per-kernel share of the serialized step
    per = defaultdict(list)
    rows = list(csv.reader(open(launches)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    H = rows[hi]
    for r in rows[hi + 1:]:
        if len(r) < len(H):
            continue
        per[r[H.index("Kernel Name")].split("(")[0].replace("void ", "")].append(float(r[H.index("Metric Value")]))
    tot = sum(sum(v) for v in per.values())
    lines += ["", "Launch list (ncu, cold-cache, serialised; compare shares):", "",
              "| kernel | launches | mean ns | share |", "|---|---|---|---|"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.0f} | {100 * sum(v) / tot:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:4])
