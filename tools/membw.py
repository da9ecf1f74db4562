"""DRAM bandwidth calibration on the GPU: pure write (zero_), read (sum), copy.

    python tools/membw.py   -> one JSON line {write_gbs, read_gbs, copy_gbs}
"""
import json

import torch


def timed(fn, reps=20):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3


n = 1 << 30  # 1 GiB per buffer (8x L2)
a = torch.empty(n // 8, dtype=torch.float64, device="cuda")
b = torch.empty(n // 8, dtype=torch.float64, device="cuda")
out = torch.empty(1, dtype=torch.float64, device="cuda")
tw = timed(lambda: a.zero_())
tr = timed(lambda: torch.sum(a, dim=0, out=out))
tc = timed(lambda: b.copy_(a))
print(json.dumps({"write_gbs": n / tw / 1e9, "read_gbs": n / tr / 1e9, "copy_gbs": 2 * n / tc / 1e9}))


def sustained(fn, nbytes, seconds):
    """Back-to-back launches for `seconds`: GB/s over the whole interval and the
    median SM clock sampled meanwhile (power-capped steady state)."""
    import subprocess
    import threading
    import time
    clocks, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            try:
                o = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-i", "0"],
                                   capture_output=True, text=True, timeout=5).stdout.strip()
                clocks.append(float(o.splitlines()[0]))
            except Exception:
                pass
            time.sleep(0.2)

    th = threading.Thread(target=sample, daemon=True)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    th.start()
    t0 = time.time()
    s.record()
    reps = 0
    while time.time() - t0 < seconds:
        for _ in range(20):
            fn()
        reps += 20
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    clocks.sort()
    return nbytes * reps / (s.elapsed_time(e) * 1e-3) / 1e9, (clocks[len(clocks) // 2] if clocks else None)


import sys  # noqa: E402

if len(sys.argv) > 2 and sys.argv[1] == "--sustained":
    secs = float(sys.argv[2])
    c, fc = sustained(lambda: b.copy_(a), 2 * n, secs)
    r, fr = sustained(lambda: torch.sum(a, dim=0, out=out), n, secs)
    print(json.dumps({"sustained_s": secs, "copy_gbs_sustained": c, "copy_sm_mhz": fc, "read_gbs_sustained": r,
                      "read_sm_mhz": fr}))
