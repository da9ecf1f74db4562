"""Device timing of single hot-path operators (CUDA events, L2 flushed between
launches): python tools/time_ops.py CONFIG [--n N] [--ops gradient,residual,...] [--reps R]

Prints one JSON line per run: median / min ms per operator.  Operators:
gradient (Q = D(U)), residual2 (R(U, Q) with Q given), residual (the public
call: gradient + residual for second-order physics), jacobian, matvec."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1204_1533_b200 import CONFIGS, LDG_K11, LineDG  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--ops", default="gradient,residual2,residual")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    case, U = cfg.build(n=a.n) if a.n else cfg.build()
    m = cfg.physics.components(cfg.dim)
    second = cfg.physics.second_order()
    stream = torch.cuda.Stream()
    ctx = LineDG(case, cfg.physics, stream=stream)
    src = cfg.source_for(case)
    if src is not None:
        ctx.set_source(src)
    Ud = torch.from_numpy(U).cuda()
    dofs = case.E * case.npe * m
    Rd = torch.empty(dofs, dtype=torch.float64, device="cuda")
    Qd = torch.empty(dofs * case.dim, dtype=torch.float64, device="cuda") if second else None
    x = torch.from_numpy(case.normal_vector(m, cfg.vector_seed)).cuda()
    y = torch.empty_like(x)
    fbuf = torch.empty(128 * 1024 * 1024, dtype=torch.int32, device="cuda")
    ops = {}
    if second:
        ops["gradient"] = lambda: ctx.gradient_residual(Ud)
        ops["residual2"] = lambda: ctx.residual_second_order(Ud, Qd)
    ops["residual"] = lambda: ctx.residual(Ud, Q_out=Qd, out=Rd)
    ops["jacobian"] = lambda: (ctx.assemble_jacobians_q(Ud, Qd) if second else ctx.assemble_jacobians(Ud))
    ops["matvec"] = lambda: (ctx.split_matvec(0.05, x, out=y) if second else ctx.spmv(LDG_K11, x, out=y))
    out = {"config": cfg.name, "n": a.n or cfg.n, "elements": case.E}
    with torch.cuda.stream(stream):
        ctx.residual(Ud, Q_out=Qd, out=Rd)
        for name in a.ops.split(","):
            if name not in ops:
                continue
            ts = []
            for r in range(a.reps + 2):
                fbuf.zero_()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                ops[name]()
                e1.record(stream)
                stream.synchronize()
                if r >= 2:
                    ts.append(e0.elapsed_time(e1))
            out[name] = {"median_ms": statistics.median(ts), "min_ms": min(ts)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
