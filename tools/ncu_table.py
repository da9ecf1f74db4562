"""Markdown table of the key ncu metrics from `ncu --page raw --csv` exports
(tools/ncu_capture.sh): time, DRAM bytes and throughput, FP64 pipe, issue
activity, occupancy, registers, launch shape and the top warp stall reasons."""
import csv
import sys

COLS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__warps_active.avg.per_cycle_active", "warps/SM"), ("launch__registers_per_thread", "regs"),
        ("launch__block_size", "block"), ("launch__grid_size", "grid")]


def rows(path):
    r = list(csv.reader(open(path)))
    h, units = r[0], r[1]
    for row in r[2:]:
        if len(row) != len(h):
            continue
        yield h, units, row


def main():
    print("| kernel | " + " | ".join(c[1] for c in COLS) + " | DRAM TB/s (% of 6.548) | top stalls |")
    print("|" + "---|" * (len(COLS) + 3))
    for path in sys.argv[1:]:
        for h, units, row in rows(path):
            name = row[h.index("Kernel Name")].split("(")[0].replace("void ", "")
            cells = []
            for key, _ in COLS:
                if key in h:
                    v, u = row[h.index(key)], units[h.index(key)]
                    cells.append(f"{v} {u}".strip())
                else:
                    cells.append("-")
            st = []
            for i, k in enumerate(h):
                if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                    try:
                        st.append((float(row[i].replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                    except ValueError:
                        pass
            tot = sum(v for v, _ in st) or 1.0
            top = ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(st, reverse=True)[:3])
            def val(key, scale):
                u = units[h.index(key)]
                x = float(row[h.index(key)].replace(",", ""))
                return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6,
                            "ns": 1e-9, "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}.get(u, scale)
            try:
                tb = (val("dram__bytes_read.sum", 1) + val("dram__bytes_write.sum", 1)) / val(
                    "gpu__time_duration.sum", 1) / 1e12
                bw = f"{tb:.2f} ({100 * tb / 6.5482:.0f} %)"
            except (ValueError, KeyError):
                bw = "-"
            print(f"| `{name}` | " + " | ".join(cells) + f" | {bw} | {top} |")


if __name__ == "__main__":
    main()
