#!/usr/bin/env python
"""Summarise ncu captures (.ncu-rep) and launch lists (--csv --log-file) into
markdown for profiles/.  Usage:
    python tools/ncu_summary.py rep1.ncu-rep [rep2 ...] [--launches launches.csv]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__warps_active.avg.per_cycle_active", "warps/SM"),
    ("launch__registers_per_thread", "regs"),
    ("launch__occupancy_limit_registers", "CTA/SM (regs)"),
    ("launch__occupancy_limit_shared_mem", "CTA/SM (smem)"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"Kernel Name": r[h.index("Kernel Name")]}
        for m, _ in METRICS:
            if m in h:
                i = h.index(m)
                d[m] = (r[i], units[i])
        res.append(d)
    return res


def short(name):
    name = name.replace("ldg::", "")
    return name[: name.find("(")] if "(" in name else name


def main(argv):
    launches = None
    reps = []
    it = iter(argv)
    for a in it:
        if a == "--launches":
            launches = next(it)
        else:
            reps.append(a)
    for rep in reps:
        print(f"### {rep.split('/')[-1]}\n")
        print("| kernel | " + " | ".join(lbl for _, lbl in METRICS) + " |")
        print("|---" * (len(METRICS) + 1) + "|")
        for d in raw(rep):
            cells = [f"{d[m][0]} {d[m][1]}".strip() if m in d else "" for m, _ in METRICS]
            print(f"| `{short(d['Kernel Name'])}` | " + " | ".join(cells) + " |")
        print()
    if launches:
        rows = list(csv.reader(open(launches)))
        hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
        h = rows[hi]
        ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
        t = defaultdict(list)
        for r in rows[hi + 1:]:
            if r[im] == "gpu__time_duration.sum":
                t[short(r[ik])].append(float(r[iv].replace(",", "")) / 1e3)
        tot = sum(sum(v) for v in t.values())
        print(f"### launch list {launches.split('/')[-1]} (cold-cache, serialised)\n")
        print("| kernel | launches | mean us | share |")
        print("|---|---|---|---|")
        for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
            print(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {100 * sum(v) / tot:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1:])
