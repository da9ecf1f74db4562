"""SPEC.md acceptance criteria that are not already covered
elsewhere (1 Table 1, 4 FD Jacobians, 5 split matvec, 6 DIRK3 order:
test_oracle_kats.py / test_time_integration.py):

  2  Poisson convergence, C11 = C22 = 0: rate of u within +-0.3 of p+1 and of
     q within +-0.3 of p (the C22 != 0 variant needs the split KKT solve the
     reference delegates to a direct solver -- out of scope, C22 = 0 here);
  3  Euler vortex convergence with RK4 on a periodic 20x15 domain: density
     error rate within +-0.3 of p+1 (GPU);
  7  free stream on the curved annulus, p in {2, 4} (test_curved_mapping.py);
  8  block-Jacobi GMRES on an implicit Navier-Stokes system: >= 3x fewer
     iterations than unpreconditioned;
  9  Jacobian reuse over >= 200 DIRK3 steps with the paper's thresholds:
     refreshes <= 10 % of Newton solves (GPU);
  10 periodic Euler vortex: total mass conserved to 1e-10 over 100 RK4 steps.
"""
import math

import numpy as np
import pytest

import scipy.sparse as sp
import scipy.sparse.linalg as spla

from paper_1204_1533_b200 import CONFIGS, LDG_K11, LDG_K12, LDG_K21, Case, _abi
from paper_1204_1533_b200.cases import Physics

from oracle.pyoracle import Oracle

G = 1.4


def node_weights(case):
    n = case.np
    m = [np.zeros(k) for k in (n, case.nq, case.nq, n * case.nq, n * case.nq, n * n, n * n, n)]
    from paper_1204_1533_b200._abi import dptr, host_lib

    host_lib().lh_basis(case.p, 1, *[dptr(a) for a in m])
    w = m[7]
    for _ in range(case.dim - 1):
        w = np.multiply.outer(w, m[7])
    return np.transpose(w, tuple(range(case.dim))[::-1]).reshape(-1)[None, :] * case.jac


# ------------------------------------------------------------------ 2
def _poisson_errors(n, p):
    """u = sin(2x) e^y on [0,1]^2, f = -lap u = 3 sin(2x) e^y, Dirichlet g = u
    (boundary function); C11 = C22 = 0 inside.  Nodal max errors of u and q."""
    case = Case.lattice(2, n, p, (1.0, 1.0, 1.0), 0.0, False, False, False, False)
    exact = lambda x, y: math.sin(2 * x) * math.exp(y)  # noqa: E731
    ora = Oracle(case, Physics(_abi.LDG_POISSON, bcs=[(t, [0.0]) for t in (1, 2, 3, 4)], c11_bd=1.0))
    for t in (1, 2, 3, 4):
        ora.set_boundary_function(t, lambda x, _t: [exact(*x)])
    X = case.coords.reshape(-1, 2)
    ora.set_source(3.0 * np.sin(2 * X[:, 0]) * np.exp(X[:, 1]))
    # linear problem: one exact Newton step, A = K11 + K12 K21 from the
    # exported triplets (checked against the oracle's split matvec)
    n = case.E * case.npe
    ora.assemble(np.zeros(n))
    k = [sp.coo_matrix((v, (i, j))).tocsr() for i, j, v in (ora.triplets(w) for w in (LDG_K11, LDG_K12, LDG_K21))]
    A = (k[0] + k[1] @ k[2]).tocsc()
    x = np.sin(np.arange(n) * 0.3)
    assert np.abs(x - 0.1 * (A @ x) - ora.split_matvec(0.1, x)).max() < 1e-10 * np.abs(A @ x).max()
    U = spla.spsolve(A, -ora.residual(np.zeros(n)))
    assert np.abs(ora.residual(U)).max() < 1e-9
    Q = ora.gradient(U).reshape(-1, 2)
    eu = np.abs(U - np.sin(2 * X[:, 0]) * np.exp(X[:, 1])).max()
    gx = 2 * np.cos(2 * X[:, 0]) * np.exp(X[:, 1])
    gy = np.sin(2 * X[:, 0]) * np.exp(X[:, 1])
    eq = max(np.abs(Q[:, 0] - gx).max(), np.abs(Q[:, 1] - gy).max())
    return eu, eq


@pytest.mark.parametrize("p", [1, 2, 3])
def test_poisson_convergence_rates(p):
    ns = (4, 8, 16)
    errs = [_poisson_errors(n, p) for n in ns]
    ru = math.log2(errs[-2][0] / errs[-1][0])
    rq = math.log2(errs[-2][1] / errs[-1][1])
    assert abs(ru - (p + 1)) <= 0.3, (p, errs, ru)
    assert abs(rq - p) <= 0.3, (p, errs, rq)


# ------------------------------------------------------------------ 8
def test_block_jacobi_effectiveness_navier_stokes():
    cfg = CONFIGS[2]
    c, U = cfg.build(n=6)
    o = Oracle(c, cfg.physics)
    o.assemble(U)
    adt = 0.05
    o.precond_build(adt)
    b = np.random.default_rng(3).standard_normal(o.n_dofs)
    _, it_pc, conv_pc, _ = o.gmres(adt, b, rtol=1e-6, maxit=3000, restart=300, precond=True)
    _, it_no, conv_no, _ = o.gmres(adt, b, rtol=1e-6, maxit=3000, restart=300, precond=False)
    assert conv_pc and conv_no
    assert it_no >= 3 * it_pc, (it_no, it_pc)


# ------------------------------------------------------------------ 10
def _vortex_prm(t, eps=5.0, x0=10.0, y0=7.5):
    return [eps, 1.5, 0.5, math.atan2(1.0, 2.0), x0, y0, 1.0, 0.5, 1.0 / G, G, t, 0.0]


def test_vortex_mass_conservation_rk4():
    case = Case.lattice(2, 6, 3, (20.0, 15.0, 1.0), 0.1, True, False, True, True, seeds=(4, 5, 6))
    U = case.fill(2, 4, _vortex_prm(0.0), 1)
    ora = Oracle(case, Physics(_abi.LDG_EULER, _abi.LDG_ROE))
    w = node_weights(case).ravel()
    mass0 = (w * U[0::4]).sum()
    for _ in range(100):
        U = ora.rk4_step(U, 0.02)
    assert abs((w * U[0::4]).sum() - mass0) <= 1e-10 * abs(mass0)


# ------------------------------------------------------------------ GPU
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1204_1533_b200.linedg import LineDG

    return torch, LineDG


@pytest.mark.gpu
def test_gpu_vortex_mass_conservation_rk4():
    torch, LineDG = _gpu()
    case = Case.lattice(2, 16, 4, (20.0, 15.0, 1.0), 0.1, True, False, True, True, seeds=(4, 5, 6))
    U = torch.from_numpy(case.fill(2, 4, _vortex_prm(0.0), 1)).cuda()
    gpu = LineDG(case, Physics(_abi.LDG_EULER, _abi.LDG_ROE))
    w = torch.from_numpy(node_weights(case).ravel()).cuda()
    mass0 = float((w * U[0::4]).sum())
    for _ in range(100):
        U = gpu.rk4_step(U, 0.02)
    assert abs(float((w * U[0::4]).sum()) - mass0) <= 1e-10 * abs(mass0)


@pytest.mark.gpu
@pytest.mark.parametrize("p", [1, 2, 3])
def test_gpu_euler_vortex_convergence(p):
    """SPEC acceptance 3: the paper's vortex (eps = 0.3, r_c = 1.5, M = 0.5,
    theta = atan(1/2)) on the periodic 20x15 domain, RK4 to t0 = sqrt(125)/10
    with dt small enough for the spatial error to dominate (temporal error
    < 1e-11).  Centred at (10, 7.5) rather than (5, 5) so that the vortex's
    tail at the periodic seam (~1e-6 at r = 7.5) stays below the finest-mesh
    error.  Meshes 16x16, 32x32, 64x64 (the oracle gives rates 1.94, 2.92,
    3.84 for p = 1, 2, 3 on the same runs)."""
    torch, LineDG = _gpu()
    t_end = math.sqrt(125.0) / 10.0
    errs = []
    for n in (16, 32, 64):
        case = Case.lattice(2, n, p, (20.0, 15.0, 1.0), 0.0, True, False, False, False)
        gpu = LineDG(case, Physics(_abi.LDG_EULER, _abi.LDG_ROE))
        U = torch.from_numpy(case.fill(2, 4, _vortex_prm(0.0, eps=0.3), 1)).cuda()
        steps = int(math.ceil(t_end * 25 * n / 8 * (p + 1)))
        for _ in range(steps):
            U = gpu.rk4_step(U, t_end / steps)
        rho = U.cpu().numpy()[0::4]
        exact = case.fill(2, 4, _vortex_prm(t_end, eps=0.3), 1)[0::4]
        errs.append(np.abs(rho - exact).max())
        gpu.close()
    rate = math.log2(errs[-2] / errs[-1])
    assert abs(rate - (p + 1)) <= 0.3, (p, errs, rate)


def _reuse_case():
    case = Case.lattice(2, 8, 3, (20.0, 15.0, 1.0), 0.1, True, False, True, True, seeds=(7, 8, 9))
    return case, Physics(_abi.LDG_EULER, _abi.LDG_ROE), case.fill(2, 4, _vortex_prm(0.0), 1)


def _count_refreshes(step, U, steps=200, dt=0.5):
    """dt = 0.5 is ~2x the RK4 stability limit on this mesh (h = 2.5, p = 3)."""
    cfg = _abi.newton_cfg(gmres_iters=5, recompute_threshold=15, max_newton=100, newton_tol=1e-8)
    refresh = 0
    for _ in range(steps):
        U, st = step(U, dt, cfg)
        refresh += st["jacobian_assemblies"]
    return refresh, 3 * steps


def test_jacobian_reuse_over_200_dirk3_steps():
    """SPEC acceptance 9 on the restated policy (the paper's thresholds:
    5 GMRES iterations per Newton update, refresh after 15 Newton updates)."""
    case, ph, U = _reuse_case()
    refresh, solves = _count_refreshes(Oracle(case, ph).dirk3_step, U)
    assert 1 <= refresh <= 0.1 * solves, (refresh, solves)


@pytest.mark.gpu
def test_gpu_jacobian_reuse_over_200_dirk3_steps():
    """SPEC acceptance 9 through the C-ABI device driver."""
    torch, LineDG = _gpu()
    case, ph, U = _reuse_case()
    gpu = LineDG(case, ph)
    refresh, solves = _count_refreshes(gpu.dirk3_step, torch.from_numpy(U).cuda())
    assert 1 <= refresh <= 0.1 * solves, (refresh, solves)
