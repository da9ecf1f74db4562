"""Per-source-line warp-stall attribution from an ncu report (needs -lineinfo).

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [N]

Prints the top-N CUDA source lines by sampled warp stalls with the dominant
stall reasons of each, and the SASS instructions that carry the samples.
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    cur_file = cur = None
    agg, src, why, sass = {}, {}, {}, {}
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 5:
            continue
        if r[0] != "":
            cur = (cur_file, int(r[0]))
            src[cur] = r[1]
            continue
        try:
            s = int(r[4])
        except ValueError:
            continue
        agg[cur] = agg.get(cur, 0) + s
        w = why.setdefault(cur, {})
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    w[h[6:]] = w.get(h[6:], 0) + int(r[i])
                except ValueError:
                    pass
        if s:
            sass.setdefault(cur, []).append((s, r[3].strip()))
    tot = sum(agg.values()) or 1
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:n]:
        reasons = sorted(why.get(k, {}).items(), key=lambda x: -x[1])[:3]
        rs = " ".join(f"{a}:{b * 100 // max(v, 1)}%" for a, b in reasons if b)
        print(f"{v / tot * 100:5.1f}% {k[0]}:{k[1]} [{rs}]  {src.get(k, '').strip()[:90]}")
        for s, ins in sorted(sass.get(k, []), reverse=True)[:2]:
            print(f"         {s / tot * 100:4.1f}%  {ins[:80]}")


if __name__ == "__main__":
    main()
