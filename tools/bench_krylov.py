"""Timing of the §8f row-1 solver pieces on one configuration (not the bench.py
contract line): block-Jacobi build, one preconditioner application, one
split matvec, and a fixed-iteration preconditioned GMRES solve.

    python tools/bench_krylov.py [--config 1] [--iters 20] [--adt 0.05]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1204_1533_b200 import CONFIGS  # noqa: E402
from paper_1204_1533_b200.linedg import LineDG  # noqa: E402


def ev_time(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--adt", type=float, default=0.05)
    ap.add_argument("--dirk-dt", type=float, default=0.01)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    case, U = cfg.build()
    g = LineDG(case, cfg.physics)
    src = cfg.source_for(case)
    if src is not None:
        g.set_source(src)
    Ud = torch.from_numpy(U).cuda()
    g.assemble_jacobians(Ud)
    b = torch.from_numpy(case.normal_vector(g.m, cfg.vector_seed)).cuda()
    ne = case.npe * g.m
    t_build_inv = t_apply_inv = None
    if ne <= 128:
        g.set_precond_mode(1)  # explicit block inverses (apply at HBM rate)
        t_build_inv = ev_time(lambda: g.precond_build(a.adt), 3)
        t_apply_inv = ev_time(lambda: g.precond_apply(b), 10)
    g.set_precond_mode(0)  # default: element-block LU (<= 128 unknowns) or line-ADI (3-D p >= 2)
    t_build = ev_time(lambda: g.precond_build(a.adt), 3)
    t_apply = ev_time(lambda: g.precond_apply(b), 10)
    t_mv = ev_time(lambda: g.split_matvec(a.adt, b), 10)
    # GMRES timed warm: the median of 5 calls after one untimed call
    # (workspace allocation and the first-call setup stay outside)
    gm = []
    for k in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, it, cv, rn = g.gmres(a.adt, b, rtol=1e-30, maxit=a.iters, restart=a.iters, precond=True)
        torch.cuda.synchronize()
        if k:
            gm.append((time.perf_counter() - t0) * 1e3)
    t_gm = float(np.median(gm))
    # one implicit DIRK3 step with the paper's Newton policy (5 GMRES / 15 Newton)
    from paper_1204_1533_b200._abi import newton_cfg
    pol = newton_cfg(gmres_iters=5, recompute_threshold=15, max_newton=100, newton_tol=1e-8)
    from paper_1204_1533_b200.linedg import SolverError
    try:
        g.dirk3_step(Ud, a.dirk_dt, pol)  # warm (Jacobian assembled, preconditioner built)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, dstats = g.dirk3_step(Ud, a.dirk_dt, pol)
        torch.cuda.synchronize()
        t_dirk = (time.perf_counter() - t0) * 1e3
    except SolverError as ex:
        t_dirk, dstats = None, {"failure": str(ex)}
    t0 = time.perf_counter()
    g.rk4_step(Ud, 1e-4)
    torch.cuda.synchronize()
    t_rk4 = (time.perf_counter() - t0) * 1e3
    if ne <= 128:
        lu_bytes = case.E * ne * ne * 8
    else:  # line-ADI factors: D (p+1)^(D-1) blocks of ((p+1) m)^2 per element
        lu_bytes = case.E * case.dim * case.NL * (case.np * g.m) ** 2 * 8
    print(json.dumps({"config": cfg.name, "dofs": g.n_dofs, "adt": a.adt,
                      "precond_build_ms": t_build, "precond_apply_ms": t_apply,
                      "precond_inverse_build_ms": t_build_inv, "precond_inverse_apply_ms": t_apply_inv,
                      "precond_apply_GBs": lu_bytes / (t_apply * 1e-3) / 1e9, "lu_bytes": lu_bytes,
                      "split_matvec_ms": t_mv, "gmres_iters": it, "gmres_ms": t_gm,
                      "gmres_ms_per_iter": t_gm / max(it, 1), "gmres_timing": "warm, median of 5 calls", "resnorm": rn,
                      "dirk3_dt": a.dirk_dt, "dirk3_step_ms": t_dirk, "dirk3_stats": dstats, "rk4_step_ms": t_rk4}))


if __name__ == "__main__":
    main()
