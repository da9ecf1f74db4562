"""Time integration (PAPER.md:641-685,
755-775): RK4, the L-stable DIRK3 with Newton + preconditioned GMRES and the
Jacobian-reuse policy.  CPU part: the oracle against SPEC known answers and
order studies.  GPU part (`-m gpu`): the device driver against the oracle.
"""
import math

import numpy as np
import pytest

from oracle.pyoracle import Oracle
from paper_1204_1533_b200 import CONFIGS, Case, Physics, _abi
from paper_1204_1533_b200._abi import newton_cfg

AL = 0.435866521508459


def tableau():
    tau2 = (1 + AL) / 2
    b1 = -(6 * AL ** 2 - 16 * AL + 1) / 4
    b2 = (6 * AL ** 2 - 20 * AL + 5) / 4
    A = np.array([[AL, 0, 0], [tau2 - AL, AL, 0], [b1, b2, AL]])
    b = np.array([b1, b2, AL])
    c = np.array([AL, tau2, 1.0])
    return A, b, c


def test_dirk3_tableau_identities():
    A, b, c = tableau()
    assert np.allclose(A.sum(axis=1), c, atol=1e-15)
    assert abs(b.sum() - 1) < 1e-15
    assert np.all(np.diag(A) == AL)
    # third order: b.c = 1/2, b.c^2 = 1/3, b.A.c = 1/6
    assert abs(b @ c - 0.5) < 1e-13 and abs(b @ c ** 2 - 1 / 3) < 1e-13 and abs(b @ A @ c - 1 / 6) < 1e-13
    # L-stability: R(z) = 1 + z b (I - zA)^-1 1 -> 0 as z -> -inf
    z = -1e6
    R = 1 + z * b @ np.linalg.solve(np.eye(3) - z * A, np.ones(3))
    assert abs(R) < 1e-5


def heat_case(p=2, n=2):
    """Heat equation u_t = Laplacian u (Poisson physics, zero Dirichlet data, no source)."""
    c = Case.lattice(2, n, p, periodic=False)
    ph = Physics(_abi.LDG_POISSON, c11_bd=1.0, bcs=[(t, [0.0]) for t in (1, 2, 3, 4)])
    xy = c.coords
    U0 = np.sin(math.pi * xy[..., 0]) * np.sin(math.pi * xy[..., 1])
    return c, ph, U0.ravel()


def integrate(o, U0, dt, T, scheme, cfg=None):
    U = U0.copy()
    for _ in range(int(round(T / dt))):
        if scheme == "rk4":
            U = o.rk4_step(U, dt)
        else:
            U, _ = o.dirk3_step(U, dt, cfg)
    return U


def test_rk4_zero_operator_and_order():
    c, ph, U0 = heat_case()
    o = Oracle(c, ph)
    assert np.array_equal(o.rk4_step(np.zeros_like(U0), 0.01), np.zeros_like(U0))  # F(0) = 0 -> bitwise
    # spectral radius of the DG heat operator here ~1250: RK4 needs dt <~ 2.2e-3
    T = 0.004
    ref = integrate(o, U0, T / 256, T, "rk4")
    errs = [np.abs(integrate(o, U0, T / m, T, "rk4") - ref).max() for m in (16, 32, 64)]
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert abs(orders[-1] - 4.0) < 0.3, orders


def test_dirk3_linear_exact_solves_one_newton_update_per_stage_and_order():
    c, ph, U0 = heat_case()
    o = Oracle(c, ph)
    n = U0.size
    # tolerance above the rounding floor of K - R (|K| ~ 20 on this stiff operator)
    exact = newton_cfg(gmres_iters=n, recompute_threshold=1000, max_newton=20, use_precond=False, newton_tol=1e-9)
    U1, st = o.dirk3_step(U0, 0.01, exact)
    assert st["newton_iters"] == 3 and st["jacobian_assemblies"] == 1  # linear: one update per stage
    T = 0.16
    ref = integrate(o, U0, 0.0025, T, "dirk3", exact)
    errs = [np.abs(integrate(o, U0, dt, T, "dirk3", exact) - ref).max() for dt in (0.04, 0.02, 0.01)]
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert abs(orders[-1] - 3.0) < 0.15, orders


def test_dirk3_free_stream_and_reuse_policy():
    c = Case.lattice(2, 3, 3, jitter=0.15, periodic=True, permute=True, rotate=True)
    o = Oracle(c, Physics(_abi.LDG_EULER))
    U = np.tile([1.0, 0.3, -0.2, 2.5], c.E * c.npe)
    U1, st = o.dirk3_step(U, 0.05, newton_cfg(newton_tol=1e-9))
    assert st["newton_iters"] == 0 and np.abs(U1 - U).max() < 1e-11  # F = 0 -> U_next = U
    # a non-trivial state: the Jacobian assembled in step 1 is reused in step 2
    cfg = CONFIGS[1]
    c2, U2 = cfg.build(n=3)
    o2 = Oracle(c2, cfg.physics)
    pol = newton_cfg(gmres_iters=5, recompute_threshold=15, max_newton=60, newton_tol=1e-8)
    U3, s1 = o2.dirk3_step(U2, 0.02, pol)
    U4, s2 = o2.dirk3_step(U3, 0.02, pol)
    assert s1["jacobian_assemblies"] == 1 and s2["jacobian_assemblies"] == 0, (s1, s2)
    assert s2["newton_iters"] >= 3
    # a tiny threshold forces reassembly inside the step
    o3 = Oracle(c2, cfg.physics)
    _, s3 = o3.dirk3_step(U2, 0.02, newton_cfg(gmres_iters=1, recompute_threshold=2, max_newton=200,
                                                newton_tol=1e-8))
    assert s3["jacobian_assemblies"] > 1, s3


def drift_case(p=2, n=2):
    """u_t = Laplacian u + S with S = x + y and time-dependent Dirichlet data
    g_D(x, t) = t (x + y) on every side: the exact solution u = t (x + y) is
    linear in space (reproduced exactly by the LDG operator) and in time, so
    RK4 and DIRK3 are exact up to rounding -- but only when every stage
    evaluates the boundary data at its own stage time."""
    c = Case.lattice(2, n, p, periodic=False)
    ph = Physics(_abi.LDG_POISSON, c11_bd=1.0, bcs=[(t, [0.0]) for t in (1, 2, 3, 4)])
    xy = c.coords.reshape(-1, 2)
    S = xy[:, 0] + xy[:, 1]
    return c, ph, S


def _drift_run(o, S, scheme, dt, steps):
    for tag in (1, 2, 3, 4):
        o.set_boundary_function(tag, lambda x, t: [t * (x[0] + x[1])])
    o.set_source(S)
    U = np.zeros_like(S)
    cfg = newton_cfg(gmres_iters=S.size, recompute_threshold=1000, max_newton=20, use_precond=False,
                     newton_tol=1e-10)
    for k in range(steps):
        if scheme == "rk4":
            U = o.rk4_step(U, dt, t=k * dt)
        else:
            U, _ = o.dirk3_step(U, dt, cfg, t=k * dt)
    return U


@pytest.mark.parametrize("scheme", ["rk4", "dirk3"])
def test_stage_times_with_time_dependent_boundary_data(scheme):
    c, ph, S = drift_case()
    dt, steps = (0.0005, 8) if scheme == "rk4" else (0.05, 4)
    U = _drift_run(Oracle(c, ph), S, scheme, dt, steps)
    exact = dt * steps * S
    assert np.abs(U - exact).max() <= 1e-9 * np.abs(exact).max(), np.abs(U - exact).max()


# ---------------------------------------------------------------- GPU parity
@pytest.mark.gpu
@pytest.mark.parametrize("scheme", ["rk4", "dirk3"])
def test_gpu_stage_times_with_time_dependent_boundary_data(scheme):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1204_1533_b200.linedg import LineDG

    c, ph, S = drift_case()
    dt, steps = (0.0005, 8) if scheme == "rk4" else (0.05, 4)
    Ug = _drift_run(LineDG(c, ph), S, scheme, dt, steps)
    Uo = _drift_run(Oracle(c, ph), S, scheme, dt, steps)
    exact = dt * steps * S
    assert np.abs(Ug - exact).max() <= 1e-9 * np.abs(exact).max()
    assert np.abs(Ug - Uo).max() <= 1e-11 * np.abs(exact).max()


# ---------------------------------------------------------------- GPU parity
@pytest.mark.gpu
@pytest.mark.parametrize("ci,n", [(1, 3), (2, 3), (0, 4)])
def test_gpu_time_steps_match_oracle(ci, n):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1204_1533_b200.linedg import LineDG

    cfg = CONFIGS[ci]
    c, U = cfg.build(n=n)
    o = Oracle(c, cfg.physics)
    g = LineDG(c, cfg.physics)
    src = cfg.source_for(c)
    if src is not None:
        o.set_source(src)
        g.set_source(src)
    dt = 0.01 if ci != 0 else 0.001
    Ur = o.rk4_step(U, dt)
    Ug = g.rk4_step(U, dt)
    assert np.abs(Ug - Ur).max() <= 1e-12 * np.abs(Ur).max()
    pol = newton_cfg(gmres_iters=5, recompute_threshold=15, max_newton=60, newton_tol=1e-8)
    Uo, so = o.dirk3_step(U, dt, pol)
    Ugd, sg = g.dirk3_step(U, dt, pol)
    assert so["newton_iters"] == sg["newton_iters"] and so["jacobian_assemblies"] == sg["jacobian_assemblies"], (so, sg)
    assert np.abs(Ugd - Uo).max() <= 1e-9 * np.abs(Uo).max()
