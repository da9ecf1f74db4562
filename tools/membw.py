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
