"""One scaled-down pass of every kernel family of a configuration (residual,
gradient, Jacobian assembly incl. K21, K11/K12/K21 products, split matvec,
block-Jacobi build/apply where supported, the host-buffer paths) for
compute-sanitizer runs (tools/sanitize.sh)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1204_1533_b200 import CONFIGS, LDG_K11, LDG_K12, LDG_K21, LineDG  # noqa: E402

ci = int(sys.argv[1])
cfg = CONFIGS[ci]
case, U = cfg.build(n=4 if cfg.dim == 2 else 2)
g = LineDG(case, cfg.physics)
m = g.m
x = case.normal_vector(m, cfg.vector_seed)
Ud, xd = torch.from_numpy(U).cuda(), torch.from_numpy(x).cuda()
Q = torch.empty(U.size * case.dim, dtype=torch.float64, device="cuda") if g.second_order else None
R = g.residual(Ud, Q_out=Q)
g.assemble_jacobians(Ud)
if Q is not None:
    g.assemble_jacobians_q(Ud, Q)
y = g.spmv(LDG_K11, xd)
if g.second_order:
    w = g.spmv(LDG_K21, xd)
    g.spmv(LDG_K12, w)
s = g.split_matvec(0.37, xd)
for order in (1, 2):
    g.set_option(1, order)
    g.spmv(LDG_K11, xd)
    g.split_matvec(0.37, xd)
try:
    g.precond_build(0.05)
    g.precond_apply(xd)
    g.gmres(0.05, xd, maxit=4)
except Exception as ex:  # configurations without a block-Jacobi preconditioner
    print("precond:", ex)
g.residual_and_assemble(U)
g.split_matvec(0.37, x)
torch.cuda.synchronize()
print("ok", float(R.abs().max()), float(s.abs().max()))
