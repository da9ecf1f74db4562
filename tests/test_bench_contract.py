"""bench.py's JSON-line contract (the driver parses it): the keys, their types
and the internal consistency of value / ms_per_step / roofline / e2e.  CPU:
the reference arm (`--impl reference`, the oracle port on the host cores) on
the small C1 configuration.  GPU: the product arm on C1 and C2 (the default
C5 line is the driver's round-end bench).
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def run_bench(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def check_common(d, steps, warmup):
    assert BASE_KEYS <= d.keys()
    assert d["n_gpus"] == 1 and d["steps"] == steps and d["warmup"] == warmup
    assert d["higher_is_better"] is True and d["scaling"] == "weak" and d["dtype"] == "f64"
    assert d["unit"] == "GDOF/s" and d["value"] > 0 and d["ms_per_step"] > 0
    dofs = d["config"]["dofs"]
    assert d["value"] == pytest.approx(dofs / (d["ms_per_step"] * 1e-3) / 1e9, rel=1e-6)
    assert d["config"]["workload"]
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]


def test_reference_arm_contract():
    d = run_bench("--impl", "reference", "--config", "0", "--steps", "3", "--warmup", "3")
    check_common(d, 3, 3)
    assert d["impl"] == "reference"
    assert d["e2e"] == {"value": d["value"], "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["cpu_baseline"]["value"] == d["value"]


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["0", "1"])
def test_product_arm_contract(cfg):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = run_bench("--config", cfg, "--steps", "3", "--warmup", "3", "--no-cpu")
    check_common_gpu = dict(d)
    check_common_gpu.setdefault("cpu_baseline", {"kind": "port", "cores": 1, "value": 1.0, "sample": "skipped"})
    check_common(check_common_gpu, 3, 3)
    assert "impl" not in d or d["impl"] != "reference"
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] == "GB/s"
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-6) and 0 < r["frac"] < 1.5
    e = d["e2e"]
    assert e["unit"] == "GDOF/s" and 0 < e["value"] < d["value"]
    n = d["config"]["dofs"] * 8
    nmv = d["config"]["matvecs"]
    assert e["h2d_bytes_per_step"] == (1 + nmv) * n and e["d2h_bytes_per_step"] == (1 + nmv) * n  # U, x up; R, y down
    assert d["gpu_launches"] > 0
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= c.keys()
    assert set(d["breakdown"]) == {"residual", "jacobian", "matvec"}
    assert r["kernel"] in d["breakdown"]
