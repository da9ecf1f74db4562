"""Space- and time-dependent boundary data (the reference's std::function g_D
/ g_N data, physics.hpp:20-31; ldg_set_boundary_function): the callback is
evaluated on the host at every boundary line end's own end node, at the t of
the call.

CPU (oracle): the SPEC known answer "single element, Dirichlet data g_D = exact
trace of a degree-p polynomial -> gradient exact to 1e-11", a
manufactured harmonic Poisson solution converging at high order through the
steady solver, time-dependent data re-evaluated when t changes.  GPU: the same
data through the C-ABI against the oracle (residual, gradient, Jacobians,
SpMVs) on Poisson, Navier-Stokes and Euler (curved cylinder) cases.
"""
import math

import numpy as np
import pytest

from paper_1204_1533_b200 import LDG_K11, LDG_K12, LDG_K21, Case, _abi
from paper_1204_1533_b200.cases import Physics, annulus_mesh

from oracle.pyoracle import Oracle

PO, NS, EU = _abi.LDG_POISSON, _abi.LDG_NAVIER_STOKES, _abi.LDG_EULER
G = 1.4


def rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    den = np.abs(b).max()
    return np.abs(a - b).max() / (den if den > 0 else 1.0)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_gradient_exact_for_polynomial_dirichlet_data(p):
    """one element, g_D the exact trace of a degree-p polynomial."""
    case = Case.lattice(2, 1, p, (1.0, 1.0, 1.0), 0.0, False, False, False, False)

    def poly(x, y):
        return 0.3 + 1.2 * x - 0.7 * y + 0.5 * x * y + (0.8 * x ** 2 - 0.4 * y ** p if p >= 2 else 0.0)

    def grad(x, y):
        return (1.2 + 0.5 * y + (1.6 * x if p >= 2 else 0.0),
                -0.7 + 0.5 * x - (0.4 * p * y ** (p - 1) if p >= 2 else 0.0))

    ora = Oracle(case, Physics(PO, bcs=[(t, [0.0]) for t in (1, 2, 3, 4)]))
    for t in (1, 2, 3, 4):
        ora.set_boundary_function(t, lambda x, _t: [poly(*x)])
    X = case.coords
    U = np.ascontiguousarray(poly(X[..., 0], X[..., 1]).reshape(-1))
    Q = ora.gradient(U).reshape(-1, 2)
    Gx, Gy = grad(X[..., 0].ravel(), X[..., 1].ravel())
    assert np.abs(Q - np.stack([Gx, Gy], axis=1)).max() < 1e-11


def _poisson_error(n, p):
    """Harmonic u = e^x sin(y) on [0,1]^2 (f = 0), Dirichlet g = u: the
    discrete steady solution's nodal max error."""
    case = Case.lattice(2, n, p, (1.0, 1.0, 1.0), 0.0, False, False, False, False)
    exact = lambda x, y: math.exp(x) * math.sin(y)  # noqa: E731
    ora = Oracle(case, Physics(PO, bcs=[(t, [0.0]) for t in (1, 2, 3, 4)], c11_bd=1.0))
    for t in (1, 2, 3, 4):
        ora.set_boundary_function(t, lambda x, _t: [exact(*x)])
    U0 = np.zeros(case.E * case.npe)
    sc = _abi.steady_cfg(dt0=1.0, n_steps=0, gmres_iters=600, gmres_rtol=1e-13, newton_tol=1e-10, max_newton=3)
    U, st = ora.steady_solve(U0, sc)
    X = case.coords
    return np.abs(U - np.vectorize(exact)(X[..., 0], X[..., 1]).ravel()).max()


def test_manufactured_poisson_converges():
    e2, e4 = _poisson_error(2, 2), _poisson_error(4, 2)
    assert e4 < e2 / 4.0 and e4 < 1e-3, (e2, e4)


def test_time_dependent_data_reevaluated():
    case = Case.lattice(2, 2, 2, (1.0, 1.0, 1.0), 0.1, False, False, True, True, seeds=(3, 4, 5))
    ora = Oracle(case, Physics(PO, bcs=[(t, [0.0]) for t in (1, 2, 3, 4)]))
    for t in (1, 2, 3, 4):
        ora.set_boundary_function(t, lambda x, tt: [tt * (x[0] + 2 * x[1])])
    U = np.sin(np.arange(case.E * case.npe) * 0.37)
    r0 = ora.residual(U, t=0.0)
    r1 = ora.residual(U, t=1.0)
    r2 = ora.residual(U, t=2.0)
    assert np.abs(r1 - r0).max() > 1e-3
    assert np.allclose(r2 - r0, 2.0 * (r1 - r0), rtol=1e-12, atol=1e-12)  # linear in the data
    ora.set_boundary_function(1, None)  # back to the constant value on tag 1
    assert not np.allclose(ora.residual(U, t=2.0), r2)


def _cases():
    def poisson():
        case = Case.lattice(2, 4, 3, (1.0, 1.0, 1.0), 0.15, False, False, True, True, seeds=(7, 8, 9))
        ph = Physics(PO, bcs=[(1, [0.0]), (2, [0.0]), (3, [0.1], _abi.LDG_BC_NEUMANN), (4, [0.0])])
        fns = {1: lambda x, t: [math.sin(3 * x[0]) + t], 2: lambda x, t: [x[1] ** 2],
               3: lambda x, t: [0.2 * x[0] - 0.1], 4: lambda x, t: [math.cos(x[1])]}
        U = np.sin(np.arange(case.E * case.npe) * 0.11)
        return case, ph, fns, U, True

    def ns():
        case = Case.lattice(2, 3, 3, (1.0, 1.0, 1.0), 0.1, False, False, True, True, seeds=(2, 3, 4))
        far = [1.0, 0.3, 0.0, 1 / (G * (G - 1)) + 0.045]

        def inflow(x, t):
            u = 0.3 + 0.05 * math.sin(math.pi * x[1])
            return [1.0, u, 0.02 * x[1], 1 / (G * (G - 1)) + 0.5 * (u * u + (0.02 * x[1]) ** 2)]
        ph = Physics(NS, mu=0.02, bcs=[(1, [0] * 4, _abi.LDG_BC_NO_SLIP_ADIABATIC), (2, far, _abi.LDG_BC_CHARACTERISTIC),
                                       (3, [0] * 4, _abi.LDG_BC_SLIP_WALL), (4, far)])
        X = case.coords
        rho = 1.0 + 0.02 * np.sin(X[..., 0])
        U = np.stack([rho, rho * 0.3, rho * 0.01, 1 / (G - 1) / G + 0.5 * rho * 0.09 + 0.01 * np.cos(X[..., 1])],
                     axis=-1)
        return case, ph, {4: inflow}, np.ascontiguousarray(U.reshape(-1)), True

    def cyl():
        v, e, b = annulus_mesh(3, 12, 0.5, 4.0, stretch=1.3)
        case = Case.custom(2, 3, v, e, b)
        case.remap_circles([(1, 0.0, 0.0, 0.5), (2, 0.0, 0.0, 4.0)])

        def far(x, t):  # slightly non-uniform far field
            u = 0.3 + 0.01 * x[1] / 4.0
            return [1.0, u, 0.0, 1 / (G * (G - 1)) + 0.5 * u * u]
        ph = Physics(EU, bcs=[(1, [0] * 4, _abi.LDG_BC_SLIP_WALL), (2, [1.0, 0.3, 0.0, 1 / (G * (G - 1)) + 0.045],
                                                                    _abi.LDG_BC_CHARACTERISTIC)])
        U = np.tile(np.array([1.0, 0.3, 0.0, 1 / (G * (G - 1)) + 0.045]), case.E * case.npe)
        return case, ph, {2: far}, U, False

    return [("poisson", poisson), ("ns-mixed", ns), ("cylinder", cyl)]


CASES = _cases()


@pytest.mark.gpu
@pytest.mark.parametrize("name,builder", CASES, ids=[c[0] for c in CASES])
def test_gpu_boundary_functions_match_oracle(name, builder):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1204_1533_b200.linedg import LineDG

    case, ph, fns, U, second = builder()
    gpu = LineDG(case, ph)
    ora = Oracle(case, ph)
    for tag, fn in fns.items():
        gpu.set_boundary_function(tag, fn)
        ora.set_boundary_function(tag, fn)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    for t in (0.0, 0.5):
        assert rel(gpu.residual(d(U), t=t).cpu().numpy(), ora.residual(U, t=t)) <= 1e-12
    sec = ph.second_order()
    if sec:
        assert rel(gpu.gradient_residual(d(U), t=0.5).cpu().numpy(), ora.gradient(U, t=0.5)) <= 1e-12
    gpu.assemble_jacobians(d(U), t=0.5)
    ora.assemble(U, t=0.5)
    for w in [LDG_K11] + ([LDG_K12, LDG_K21] if sec else []):
        r0, c0, v0 = ora.export_blocks(w)
        r1, c1, v1 = gpu.export_blocks(w)
        assert np.array_equal(r0, r1) and np.array_equal(c0, c1)
        assert rel(v1, v0) <= 1e-12
    x = case.normal_vector(gpu.m, 3)
    assert rel(gpu.split_matvec(0.1, d(x)).cpu().numpy(), ora.split_matvec(0.1, x)) <= 1e-12
