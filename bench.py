#!/usr/bin/env python
"""Benchmark of the Line-DG hot path on B200 (BASELINE.json metric).

One step = one pass of the hot path over the configuration's synthetic input,
fp64: the residual R(U) (second-order physics: Q = D(U), then R(U, Q)), the
analytic Jacobian assembly at U (sharing that Q, as a Newton step does), and
NMV matvecs with the assembled Jacobian on seeded N(0,1) vectors -- the split
matvec (I - adt (K11 + K12 K21)) v that GMRES applies for second-order physics,
the K11 block-SpMV for first-order physics.  The default workload is the
largest single-GPU configuration, BASELINE.json config 5 (3-D Navier-Stokes
p=4 48^3, 69 M DOFs, 164 GB Jacobian store): "full residual, Jacobian assembly
and 30 block-SpMVs on seeded N(0,1) vectors" (NMV = 30; other configs NMV = 1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

value      = DOFs processed per second through the whole step (all ranks), GDOF/s,
             inputs resident in HBM, L2 flushed (512 MB write + read) between steps
             (every C3-C5 operand is also larger than the 126 MB L2).
e2e        = the same step through the reference-facing host-buffer C-ABI
             (ldg_residual_assemble_host: one upload of U, R downloaded; then NMV
             ldg_split_matvec_host / ldg_bsr_spmv_host calls, v up and y down each),
             asynchronous mode + ldg_synchronize, all transfers inside the timed region.
roofline   = the step's dominant kernel family: algorithmic bytes per launch / mean
             CUDA-event duration vs the measured HBM copy bandwidth.
cpu_baseline = the CPU oracle (oracle/, a port of the reference algorithm; the
             reference's own hot-path sources do not exist) on this host: a
             cost-proportional element subset of the same step, extrapolated
             linearly to the full mesh, all host threads, plus a 1-thread figure.
--impl reference runs only that CPU implementation.
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
    ns11 = D * p + 1 + 2 * D
    ns12 = D * p + 1 + D
    r12 = m - 1 if m > 1 else 1
    K11 = 8 * N * ns11 * m * m
    K12 = 8 * N * ns12 * r12 * m * D
    K21 = 8 * N * ns12 * D
    if not second:
        out["residual"] = 2 * U + 8 * met * E + conn
    else:
        # gradient pass (Q out) + residual pass (U, Q in, R out)
        out["residual"] = (U + 8 * met * E + conn + U * D) + (U + U * D + 8 * met * E + conn + U)
    out["jacobian"] = K11 + U + 8 * met * E + conn
    if second:
        # K12 = dR/dQ re-assembled with K11 every step (K21 is U-independent,
        # assembled once), plus the gradient Q read
        out["jacobian"] += K12 + U * D
        # split matvec: K21 pass (v in, w out), then K11 v + K12 w and the axpy
        out["matvec"] = (K21 + U + U * D + conn) + (K11 + K12 + U + U * D + U + conn)
    else:
        out["matvec"] = K11 + 2 * U + conn
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
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_cpu(cfg, case, U, xs, nmv, adt, steps, budget_s=20.0, threads=None, frac=None):
    """The oracle (CPU port of the reference algorithm) on a cost-proportional
    element subset of the step (lo_time_sample), extrapolated linearly to the
    full mesh: returns (full-step seconds per sample, threads, subset size)."""
    from oracle.pyoracle import Oracle  # CPU baseline leg only

    threads = threads or Oracle.max_threads()
    ora = Oracle(case, cfg.physics)
    src = cfg.source_for(case)
    if src is not None:
        ora.set_source(src)
    # subset size: a first small probe, then sized so one sample takes ~budget/steps
    n = max(1, min(case.E, case.E // (frac or 512)))
    elems = np.arange(case.E, dtype=np.int32)
    probe = ora.time_sample(U, xs[0], adt, nmv, elems[:n], threads, reps=1).sum()
    if frac is None:
        want = max(0.5, budget_s / max(1, steps))
        n = int(min(case.E, max(n, n * want / max(probe, 1e-6))))
    out = []
    t0 = time.perf_counter()
    for _ in range(max(1, steps)):
        secs = ora.time_sample(U, xs[0], adt, nmv, elems[:n], threads, reps=1)
        out.append(float(secs.sum()) * case.E / n)
        if time.perf_counter() - t0 > budget_s:
            break
    ora.close() if hasattr(ora, "close") else None
    return out, threads, n


# ---------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4,
                    help="BASELINE.json config index (4 = 3-D Navier-Stokes p=4 48^3, the largest single-GPU config)")
    ap.add_argument("--matvecs", type=int, default=None, help="matvecs per step (default: 30 for config 4, else 1)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer end-to-end leg")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = CONFIGS[args.config]
    m = cfg.physics.components(cfg.dim)
    second = cfg.physics.second_order()
    nmv = args.matvecs if args.matvecs is not None else (30 if args.config == 4 else 1)
    nvec = max(1, min(3, nmv))
    ADT = 0.05
    mv_name = "split matvec (I - adt(K11 + K12 K21)) v" if second else "K11 block-SpMV"
    metric = "residual GDOF/s, Jacobian assembly + block-SpMV GB/s (fp64), % HBM roofline, 1 B200"
    workload = {"workload": cfg.name, "config_index": args.config, "elements": cfg.n ** cfg.dim,
                "p": cfg.p, "dofs": cfg.dofs(),
                "step": f"residual + Jacobian assembly (one shared Q = D(U)) + {nmv} x {mv_name}",
                "matvecs": nmv, "matvec_vectors": f"{nvec} seeded N(0,1) vectors, cycled; alpha_dt = {ADT}",
                "l2": "flushed between steps (512 MB write + 512 MB read); C3-C5 operands also exceed L2",
                "parallelism": "replicas" if world > 1 else "1 GPU"}

    if args.impl == "reference":
        if rank != 0:
            return
        case, U = cfg.build()
        xs = [case.normal_vector(m, cfg.vector_seed + k) for k in range(nvec)]
        warm, _, _ = run_cpu(cfg, case, U, xs, nmv, ADT, max(1, min(args.warmup, 1)), budget_s=10.0)
        times, threads, n = run_cpu(cfg, case, U, xs, nmv, ADT, args.steps, budget_s=max(30.0, args.cpu_budget))
        t = statistics.median(times)
        dofs = case.E * case.npe * m
        val = dofs / t / 1e9
        line = {"metric": metric, "impl": "reference", "value": val, "unit": "GDOF/s", "n_gpus": args.gpus,
                "steps": len(times), "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded, BASELINE.json config shapes)", "config": workload,
                "cpu_baseline": {"value": val, "unit": "GDOF/s", "cores": threads, "kind": "port",
                                 "cpu": cpu_model(),
                                 "sample": f"{cfg.name} step on {n} of {case.E} elements per sample (oracle, "
                                           f"OpenMP), extrapolated linearly to the full mesh; median of "
                                           f"{len(times)}"},
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
    xs_h = [case.normal_vector(m, cfg.vector_seed + k) for k in range(nvec)]
    N = case.E * case.npe
    dofs = N * m
    stream = torch.cuda.Stream()
    ctx = LineDG(case, cfg.physics, stream=stream)
    src = cfg.source_for(case)
    if src is not None:
        ctx.set_source(src)
    Ud = torch.from_numpy(U).cuda()
    xs = [torch.from_numpy(x).cuda() for x in xs_h]
    Rd = torch.empty(dofs, dtype=torch.float64, device="cuda")
    Qd = torch.empty(dofs * case.dim, dtype=torch.float64, device="cuda") if second else None
    ys = [torch.empty(dofs, dtype=torch.float64, device="cuda") for _ in range(min(2, nmv))]
    # L2 flush between steps: write 512 MB (> 126 MB L2), then read another
    # 512 MB so the lines left in L2 are clean (no write-back lands in the
    # next timed kernel).
    fbuf = torch.empty(128 * 1024 * 1024, dtype=torch.int32, device="cuda")
    rbuf = torch.ones(128 * 1024 * 1024, dtype=torch.int32, device="cuda")
    fsink = torch.empty((), dtype=torch.int64, device="cuda")

    def flush():
        fbuf.zero_()
        torch.sum(rbuf, dim=0, out=fsink)

    def op_residual():
        ctx.residual(Ud, Q_out=Qd, out=Rd)

    def op_jacobian():
        if second:
            ctx.assemble_jacobians_q(Ud, Qd)
        else:
            ctx.assemble_jacobians(Ud)

    def op_matvecs():
        for k in range(nmv):
            if second:
                ctx.split_matvec(ADT, xs[k % nvec], out=ys[k % 2])
            else:
                ctx.spmv(LDG_K11, xs[k % nvec], out=ys[k % 2])

    ops = [op_residual, op_jacobian, op_matvecs]
    torch.cuda.synchronize()
    ctx.set_sync_errors(False)
    with torch.cuda.stream(stream):
        for _ in range(max(1, args.warmup)):
            flush()
            for op in ops:
                op()
    ctx.synchronize()
    # Each op of the step is captured once as a CUDA graph and replayed; the
    # event pairs around the replays time each op on the launching stream.
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
            flush()
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
    # kernels per step: counted by the library over one (uncaptured) step
    n0 = ctx.kernel_launches()
    with torch.cuda.stream(stream):
        for op in ops:
            op()
    ctx.synchronize()
    launches = (ctx.kernel_launches() - n0) * args.steps
    t_res = statistics.median(p[0] for p in per)
    t_jac = statistics.median(p[1] for p in per)
    t_mvs = statistics.median(p[2] for p in per)
    ms = statistics.median(p[3] for p in per)
    ms = max_over_ranks(ms)
    value = replica_throughput(dofs, world, ms)

    # ---- end to end through the host-buffer C-ABI (pinned host memory)
    e2e = None
    if not args.no_e2e:
        Uh = torch.from_numpy(U).pin_memory().numpy()
        xh = [torch.from_numpy(x).pin_memory().numpy() for x in xs_h]
        Rh = torch.empty(dofs, dtype=torch.float64).pin_memory().numpy()
        yh = [torch.empty(dofs, dtype=torch.float64).pin_memory().numpy() for _ in range(min(2, nmv))]
        ctx.set_sync_errors(False)
        e2e_times = []
        for k in range(args.warmup + args.steps):
            with torch.cuda.stream(stream):
                flush()
            torch.cuda.synchronize()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            ctx.residual_and_assemble(Uh, out=Rh)
            for j in range(nmv):
                if second:
                    ctx.split_matvec(ADT, xh[j % nvec], out=yh[j % 2])
                else:
                    ctx.spmv(LDG_K11, xh[j % nvec], out=yh[j % 2])
            ctx.synchronize()
            t1.record(stream)
            torch.cuda.synchronize()
            if k >= args.warmup:
                e2e_times.append(t0.elapsed_time(t1))
        ctx.set_sync_errors(True)
        e2e_ms = max_over_ranks(statistics.median(e2e_times))
        e2e = {"value": world * dofs / (e2e_ms * 1e-3) / 1e9, "unit": "GDOF/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": 8 * dofs * (1 + nmv), "d2h_bytes_per_step": 8 * dofs * (1 + nmv),
               "path": "ldg_residual_assemble_host + NMV x " +
                       ("ldg_split_matvec_host" if second else "ldg_bsr_spmv_host") + " (pinned, asynchronous)"}

    # ---- roofline of the dominant kernel family
    hbm, peak_src = peaks()
    by = sizes(cfg, case, m)
    kern = {"residual": t_res, "jacobian": t_jac, "matvec": t_mvs / nmv}
    share = {"residual": t_res / ms, "jacobian": t_jac / ms, "matvec": t_mvs / ms}
    dom = max(share, key=share.get)
    breakdown = {}
    for name, tms in kern.items():
        gbs = by[name] / (tms * 1e-3) / 1e9
        breakdown[name] = {"ms_per_launch": tms, "launches_per_step": nmv if name == "matvec" else 1,
                           "share_of_step": share[name], "GB/s": gbs, "frac_hbm": gbs / hbm,
                           "alg_bytes": by[name]}
    breakdown["residual"]["GDOF/s"] = dofs / (t_res * 1e-3) / 1e9
    p64, p64_src = fp64_peak()
    fl = flops(args.config, case)
    if fl is not None:
        fl = {"residual": fl["residual"], "jacobian": fl["jacobian"], "matvec": fl["spmv"]}
        for name, tms in kern.items():
            tf = fl[name] / (tms * 1e-3) / 1e12
            breakdown[name].update({"alg_flops": fl[name], "TFLOP/s": tf, "frac_fp64": tf / p64,
                                    "frac_roofline": max(breakdown[name]["frac_hbm"], tf / p64)})
    achieved = by[dom] / (kern[dom] * 1e-3) / 1e9
    line = {"metric": metric, "value": value, "unit": "GDOF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json config shapes)",
            "config": workload,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": None,
                         "traffic_note": "ncu dram__bytes_read+write per launch: profiles/ (not measured in-run)",
                         "peak_source": peak_src},
            "breakdown": breakdown, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
            "jacobian_store_bytes": ctx.jacobian_bytes()}
    if rank == 0 and world == 1 and not args.no_cpu:
        ctx.close()
        del Ud, xs, Rd, Qd, ys
        times, threads, n = run_cpu(cfg, case, U, xs_h, nmv, ADT, 3, args.cpu_budget)
        t1c, _, n1 = run_cpu(cfg, case, U, xs_h, nmv, ADT, 1, args.cpu_budget / 4, threads=1,
                             frac=max(1, case.E // max(1, n // max(1, threads))))
        line["cpu_baseline"] = {
            "value": dofs / statistics.median(times) / 1e9, "unit": "GDOF/s", "cores": threads, "kind": "port",
            "cpu": cpu_model(), "value_1core": dofs / t1c[0] / 1e9,
            "sample": f"{cfg.name} step on {n} of {case.E} elements ({threads} threads; 1-thread figure on {n1}), "
                      f"oracle lo_time_sample, extrapolated linearly to the full mesh; median of {len(times)}"}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
