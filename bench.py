#!/usr/bin/env python
"""Benchmark of the Line-DG hot path on B200 (BASELINE.json metric).

One step = one pass of the hot path over the configuration's synthetic input:
residual (GDOF/s) + analytic Jacobian assembly + block-SpMV on a seeded N(0,1)
vector (BASELINE.json config 2: "residual + Jacobian + block-SpMV"), fp64.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1] [--impl ours|reference]

value      = DOFs processed per second through the whole step (all ranks), GDOF/s,
             inputs resident in HBM, L2 flushed (512 MB write) between steps.
e2e        = same metric through the reference-facing host-buffer C-ABI calls
             (ldg_residual_host, ldg_jacobian_assemble_host, ldg_bsr_spmv_host,
             asynchronous mode + ldg_synchronize): H2D of U (twice: residual and
             assembly inputs) and x, D2H of R and y, all inside the timed region.
roofline   = the step's dominant kernel: algorithmic bytes per launch / mean
             CUDA-event duration vs the measured HBM copy bandwidth.
cpu_baseline = the CPU oracle (oracle/, a port of the reference algorithm;
             the reference's own hot-path sources do not exist) on this host.
--impl reference runs only that CPU implementation (all host threads).
Multi-GPU: the north star keeps the path on one GPU ("nothing across GPUs"),
so N > 1 runs N independent replicas (weak scaling, no collective).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1204_1533_b200 import CONFIGS, LDG_K11, LDG_K12, LDG_K21  # noqa: E402


# ---------------------------------------------------------------- helpers
def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def fp64_peak():
    """Measured FP64 FMA peak (tools/fp64_peak.cu on this pool's B200, written to
    profiles/fp64_peak.json), else the B200 datasheet figure."""
    path = os.path.join(ROOT, "profiles", "fp64_peak.json")
    try:
        with open(path) as f:
            return float(json.load(f)["fp64_tflops"]), "measured (profiles/fp64_peak.json, tools/fp64_peak.cu)"
    except Exception:
        return 40.0, "nominal (B200 datasheet 40 TFLOP/s FP64)"


def flops(index, case):
    """Algorithmic FP64 flops per launch (profiles/flops.json, tools/flop_model.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "flops.json")) as f:
            fm = json.load(f)[f"config{index}"]
    except Exception:
        return None
    return {k: fm[k] * case.E for k in ("residual", "jacobian", "spmv")}


def sizes(cfg, case, m):
    """Algorithmic bytes per launch (adapted to this store:
    no column-index stream)."""
    D, E, npe = case.dim, case.E, case.npe
    NL, nq, p = case.NL, case.nq, case.p
    N = E * npe
    met = D * NL * nq * D + 2 * D * NL * D + npe
    conn = 8 * 2 * D * E + 4 * E
    U = 8 * N * m
    out = {}
    second = cfg.physics.second_order()
    if not second:
        out["residual"] = 2 * U + 8 * met * E + conn
    else:
        out["gradient"] = U + 8 * met * E + conn + U * D
        out["residual"] = U + U * D + 8 * met * E + conn + U
    ns11 = D * p + 1 + 2 * D
    out["jacobian"] = 8 * N * ns11 * m * m + U + 8 * met * E + conn
    if second:
        # K12 = dR/dQ is re-assembled with K11 every step (K21 is U-independent,
        # assembled once): ns12 node-columns of r12 x m*D blocks per row
        # (Navier-Stokes drops the density row), plus the gradient Q read.
        ns12 = D * p + 1 + D
        r12 = m - 1 if m > 1 else 1
        out["jacobian"] += 8 * N * ns12 * r12 * m * D + U * D
    out["spmv"] = 8 * N * ns11 * m * m + 2 * U + conn
    return out


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()
        time.sleep(0.15)

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 6:
                self.rows.append(parts)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "", 1).isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "", 1).isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def max_over_ranks(x: float, device: str = "cuda") -> float:
    """Max of a per-rank time over all ranks (NCCL on the GPU run, gloo in tests)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_throughput(dofs_per_rank: int, world: int, ms_max: float) -> float:
    """Whole-job GDOF/s of N independent replicas timed as the max over ranks."""
    return world * dofs_per_rank / (ms_max * 1e-3) / 1e9


def _kernels_per_step(ctx, step, stream, torch):
    """Kernel launches the library issues for one step (its own counter)."""
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    n0 = ctx.kernel_launches()
    with torch.cuda.stream(stream):
        step(ev)
    stream.synchronize()
    return ctx.kernel_launches() - n0


# ---------------------------------------------------------------- CPU leg
def cpu_step_fn(cfg, case, U, x):
    from oracle.pyoracle import Oracle  # CPU baseline leg only

    ora = Oracle(case, cfg.physics)
    src = cfg.source_for(case)
    if src is not None:
        ora.set_source(src)

    def step():
        ora.residual(U)
        ora.assemble(U)
        ora.spmv(LDG_K11, x)
    return ora, step


def run_cpu(cfg, case, U, x, steps, warmup, budget_s=20.0):
    from oracle.pyoracle import Oracle

    threads = Oracle.max_threads()
    Oracle.set_threads(threads)
    _, step = cpu_step_fn(cfg, case, U, x)
    t0 = time.perf_counter()
    for _ in range(max(1, warmup)):
        step()
        if time.perf_counter() - t0 > budget_s / 2:
            break
    times = []
    for _ in range(max(1, steps)):
        t = time.perf_counter()
        step()
        times.append(time.perf_counter() - t)
        if sum(times) > budget_s:
            break
    dofs = case.E * case.npe * cfg.physics.components(case.dim)
    return dofs, times, threads


# ---------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=1, help="BASELINE.json config index (1 = 2-D Euler p=4 128^2)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = CONFIGS[args.config]
    m = cfg.physics.components(cfg.dim)
    workload = {"workload": cfg.name, "config_index": args.config, "elements": cfg.n ** cfg.dim,
                "p": cfg.p, "dofs": cfg.dofs(), "step": "residual + Jacobian assembly + K11 block-SpMV",
                "l2": "flushed between steps (512 MB write + 512 MB read)", "parallelism": "replicas" if world > 1 else "1 GPU"}

    if args.impl == "reference":
        if rank != 0:
            return
        case, U = cfg.build()
        x = case.normal_vector(m, cfg.vector_seed)
        dofs, times, threads = run_cpu(cfg, case, U, x, args.steps, args.warmup, budget_s=max(30.0, args.cpu_budget))
        t = statistics.mean(times)
        val = dofs / t / 1e9
        line = {"metric": "residual GDOF/s, Jacobian assembly + block-SpMV GB/s (fp64), % HBM roofline, 1 B200",
                "impl": "reference", "value": val, "unit": "GDOF/s", "n_gpus": args.gpus, "steps": len(times),
                "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json config shapes)",
                "config": workload,
                "cpu_baseline": {"value": val, "unit": "GDOF/s", "cores": threads, "kind": "port",
                                 "sample": f"full {cfg.name} step (all {case.E} elements) x {len(times)}"},
                "e2e": {"value": val, "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch

    from paper_1204_1533_b200 import LineDG

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    case, U = cfg.build()
    x = case.normal_vector(m, cfg.vector_seed)
    N = case.E * case.npe
    dofs = N * m
    stream = torch.cuda.Stream()
    ctx = LineDG(case, cfg.physics, stream=stream)
    src = cfg.source_for(case)
    if src is not None:
        ctx.set_source(src)
    Ud = torch.from_numpy(U).cuda()
    xd = torch.from_numpy(x).cuda()
    # L2 flush between steps: write 512 MB (> 126 MB L2), then read another
    # 512 MB so the lines left in L2 are clean (no write-back lands in the
    # next timed kernel).
    fbuf = torch.empty(128 * 1024 * 1024, dtype=torch.int32, device="cuda")
    rbuf = torch.ones(128 * 1024 * 1024, dtype=torch.int32, device="cuda")
    fsink = torch.empty((), dtype=torch.int64, device="cuda")

    class _Flush:
        @staticmethod
        def zero_():
            fbuf.zero_()
            torch.sum(rbuf, dim=0, out=fsink)

    flush = _Flush()
    torch.cuda.synchronize()
    ctx.set_sync_errors(False)

    def step(ev):
        ev[0].record(stream)
        ctx.residual(Ud)
        ev[1].record(stream)
        ctx.assemble_jacobians(Ud)
        ev[2].record(stream)
        ctx.spmv(LDG_K11, xd)
        ev[3].record(stream)

    with torch.cuda.stream(stream):
        for _ in range(max(1, args.warmup)):
            flush.zero_()
            step([torch.cuda.Event(enable_timing=True) for _ in range(4)])
    ctx.synchronize()
    # Each op of the step is captured once as a CUDA graph and replayed; the
    # event pairs around the replays time each kernel on the launching
    # stream.  The 512 MB L2-flush kernel ahead of every step keeps the host
    # ahead of the GPU, so no host launch gap falls inside a timed interval.
    ops = [lambda: ctx.residual(Ud), lambda: ctx.assemble_jacobians(Ud), lambda: ctx.spmv(LDG_K11, xd)]
    graphs = []
    for op in ops:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            op()
        graphs.append(g)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    sampler = ClockSampler(local)
    sampler.start()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for k in range(args.steps):
            flush.zero_()
            evs[k][0].record(stream)
            for i, g in enumerate(graphs):
                g.replay()
                evs[k][i + 1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = sampler.stop()
    ctx.synchronize()  # surfaces any physical-state failure of the timed steps
    per = [(e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3]), e[0].elapsed_time(e[3]))
           for e in evs]
    # kernels per step: counted by the library while capturing the step
    n_per_step = _kernels_per_step(ctx, step, stream, torch)
    launches = n_per_step * args.steps
    t_res = statistics.mean(p[0] for p in per)
    t_jac = statistics.mean(p[1] for p in per)
    t_spv = statistics.mean(p[2] for p in per)
    ms = statistics.mean(p[3] for p in per)
    ms = max_over_ranks(ms)
    value = replica_throughput(dofs, world, ms)

    # ---- end to end through the host-buffer C-ABI (pinned host memory)
    Uh = torch.from_numpy(U).pin_memory().numpy()
    xh = torch.from_numpy(x).pin_memory().numpy()
    Rh = torch.empty(U.size, dtype=torch.float64).pin_memory().numpy()  # pinned result buffers
    yh = torch.empty(x.size, dtype=torch.float64).pin_memory().numpy()
    # asynchronous host-buffer calls (ldg_set_sync_errors(ctx, 0)): uploads and
    # downloads run on the context's copy streams and overlap the kernels and
    # each other; ldg_synchronize joins them (results valid after it).
    ctx.set_sync_errors(False)
    e2e_times = []
    torch.cuda.set_stream(stream)
    for k in range(args.warmup + args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        ctx.residual(Uh, out=Rh)
        ctx.assemble_jacobians(Uh)
        ctx.spmv(LDG_K11, xh, out=yh)
        ctx.synchronize()
        t1.record(stream)
        torch.cuda.synchronize()
        if k >= args.warmup:
            e2e_times.append(t0.elapsed_time(t1))
    ctx.set_sync_errors(True)
    e2e_ms = statistics.mean(e2e_times)
    e2e_ms = max_over_ranks(e2e_ms)

    # ---- roofline of the dominant kernel
    hbm, peak_src = peaks()
    by = sizes(cfg, case, m)
    kern = {"residual": t_res, "jacobian": t_jac, "spmv": t_spv}
    dom = max(kern, key=kern.get)
    breakdown = {}
    for name, tms in kern.items():
        b = by[name] if name != "residual" else by["residual"] + by.get("gradient", 0)
        gbs = b / (tms * 1e-3) / 1e9
        breakdown[name] = {"ms": tms, "GB/s": gbs, "frac_hbm": gbs / hbm, "alg_bytes": b}
    breakdown["residual"]["GDOF/s"] = dofs / (t_res * 1e-3) / 1e9
    # FP64 side of the roofline (fraction = max(bytes/BW, flops/P_fp64))
    p64, p64_src = fp64_peak()
    fl = flops(args.config, case)
    if fl is not None:
        for name, tms in kern.items():
            tf = fl[name] / (tms * 1e-3) / 1e12
            breakdown[name].update({"alg_flops": fl[name], "TFLOP/s": tf, "frac_fp64": tf / p64,
                                    "frac_roofline": max(breakdown[name]["frac_hbm"], tf / p64)})
    bdom = by[dom] if dom != "residual" else by["residual"] + by.get("gradient", 0)
    achieved = bdom / (kern[dom] * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                traffic = json.load(f).get(f"config{args.config}", {}).get(dom)
        except Exception:
            traffic = None

    line = {"metric": "residual GDOF/s, Jacobian assembly + block-SpMV GB/s (fp64), % HBM roofline, 1 B200",
            "value": value, "unit": "GDOF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE.json config shapes)", "config": workload,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic, "peak_source": peak_src,
                         "fp64": None if fl is None else {
                             "flops": fl[dom], "achieved_tflops": fl[dom] / (kern[dom] * 1e-3) / 1e12,
                             "peak_tflops": p64, "frac": fl[dom] / (kern[dom] * 1e-3) / 1e12 / p64,
                             "peak_source": p64_src}},
            "breakdown": breakdown,
            "e2e": {"value": world * dofs / (e2e_ms * 1e-3) / 1e9, "unit": "GDOF/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": 3 * 8 * dofs, "d2h_bytes_per_step": 2 * 8 * dofs},
            "gpu_launches": launches, "clocks": clocks,
            "jacobian_store_bytes": ctx.jacobian_bytes()}
    if rank == 0 and world == 1 and not args.no_cpu:
        cd, times, threads = run_cpu(cfg, case, U, x, max(2, min(args.steps, 10)), 1, args.cpu_budget)
        line["cpu_baseline"] = {"value": cd / statistics.mean(times) / 1e9, "unit": "GDOF/s", "cores": threads,
                                "kind": "port", "sample": f"full {cfg.name} step x {len(times)} (oracle, OpenMP)"}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
