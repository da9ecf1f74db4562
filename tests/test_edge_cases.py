"""Edge cases of the hot path: the smallest and most boundary-dominated
inputs (a single element whose every face is a boundary, one-element-wide
strips, p = 1), the largest supported degree, and refused inputs (empty mesh,
unsupported degree, inverted element) -- on the oracle (CPU) and through the
C-ABI on the GPU against it (values <= 1e-12 normwise, patterns bit-exact).
"""
import numpy as np
import pytest

from paper_1204_1533_b200 import LDG_K11, LDG_K12, LDG_K21, Case, _abi
from paper_1204_1533_b200.cases import Physics

from oracle.pyoracle import Oracle

G = 1.4
EU, NS, PO = _abi.LDG_EULER, _abi.LDG_NAVIER_STOKES, _abi.LDG_POISSON


def rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    den = np.abs(b).max()
    return np.abs(a - b).max() / (den if den > 0 else 1.0)


def state(case, kind, seed=3):
    rng = np.random.default_rng(seed)
    x = case.coords
    if kind == PO:
        return np.ascontiguousarray(np.sin(2.0 * x[..., 0] + x[..., 1]).reshape(-1) + 0.01 * rng.standard_normal(
            case.E * case.npe))
    D = case.dim
    rho = 1.0 + 0.05 * np.sin(x[..., 0] + 0.5)
    vel = [0.3 + 0.05 * np.cos(x[..., d]) for d in range(D)]
    p = 1 / G + 0.02 * np.sin(x[..., D - 1])
    E = p / (G - 1) + 0.5 * rho * sum(v * v for v in vel)
    return np.ascontiguousarray(np.stack([rho] + [rho * v for v in vel] + [E], axis=-1).reshape(-1))


def dirichlet_all(case, kind):
    D = case.dim
    m = 1 if kind == PO else D + 2
    g = [0.2] if kind == PO else [1.0, 0.3] + [0.1] * (D - 1) + [1 / (G * (G - 1)) + 0.5 * (0.09 + 0.01 * (D - 1))]
    return [(t, g[:m]) for t in range(1, 2 * D + 1)]


CASES = [  # name, dim, nx (elements per direction; strips via custom), p, physics
    ("single-2d-poisson-p1", 2, 1, 1, PO), ("single-2d-euler-p4", 2, 1, 4, EU), ("single-2d-ns-p2", 2, 1, 2, NS),
    ("single-3d-euler-p1", 3, 1, 1, EU), ("single-3d-ns-p3", 3, 1, 3, NS), ("single-3d-poisson-p4", 3, 1, 4, PO),
    ("strip-2d-euler-p3", 2, "strip", 3, EU), ("strip-2d-ns-p4", 2, "strip", 4, NS),
]


def build(dim, nx, p, kind):
    if nx == "strip":  # 1 x 7 elements, jitter-free: one-element-wide, every element touches two boundaries
        n = 7
        verts = np.array([[i / n, j * 0.3] for j in range(2) for i in range(n + 1)])
        elems = np.array([[i, i + 1, n + 2 + i, n + 1 + i] for i in range(n)], dtype=np.int32)
        btags = [[e, 0, 1] for e in range(n)] + [[e, 2, 3] for e in range(n)] + [[0, 3, 4], [n - 1, 1, 2]]
        case = Case.custom(2, p, verts, elems, btags)
    else:
        case = Case.lattice(dim, nx, p, (1.0, 1.0, 1.0), 0.0, False, False, False, True, seeds=(5, 6, 7))
    mu = 0.05 if kind == NS else 0.0
    ph = Physics(kind, mu=mu, bcs=dirichlet_all(case, kind))
    return case, ph, state(case, kind)


@pytest.mark.parametrize("name,dim,nx,p,kind", CASES, ids=[c[0] for c in CASES])
def test_oracle_edge_case_properties(name, dim, nx, p, kind):
    """Analytic Jacobians equal finite differences on the boundary-dominated
    meshes (every line end of the single element is a boundary end)."""
    case, ph, U = build(dim, nx, p, kind)
    ora = Oracle(case, ph)
    assert np.isfinite(ora.residual(U)).all()
    if case.E * case.npe * (1 if kind == PO else dim + 2) > 600:
        pytest.skip("dense FD check sized for small cases")
    ora.assemble(U)
    second = ph.second_order()
    Q = ora.gradient(U) if second else None
    for w in [LDG_K11] + ([LDG_K12, LDG_K21] if second else []):
        A = ora.dense(w)
        F = ora.fd_dense(w, U, Q)
        assert rel(A, F) < 1e-6, (w, rel(A, F))


def test_refused_inputs_oracle():
    with pytest.raises(RuntimeError, match="no elements"):
        empty = Case.custom(2, 2, np.zeros((0, 2)), np.zeros((0, 4), np.int32))
        Oracle(empty, Physics(EU))
    # clockwise (inverted) element: refused as a config_error (mesh.cpp:19-29)
    from paper_1204_1533_b200.linedg import ConfigError

    with pytest.raises(ConfigError, match="counter-clockwise|inverted"):
        Case.custom(2, 2, np.array([[0, 0], [0, 1], [1, 1], [1, 0]], float), np.array([[0, 1, 2, 3]], np.int32))


@pytest.mark.gpu
@pytest.mark.parametrize("name,dim,nx,p,kind", CASES, ids=[c[0] for c in CASES])
def test_gpu_edge_cases_match_oracle(name, dim, nx, p, kind):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1204_1533_b200.linedg import LineDG

    case, ph, U = build(dim, nx, p, kind)
    gpu = LineDG(case, ph)
    ora = Oracle(case, ph)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    assert rel(gpu.residual(d(U)).cpu().numpy(), ora.residual(U)) <= 1e-12
    gpu.assemble_jacobians(d(U))
    ora.assemble(U)
    second = ph.second_order()
    for w in [LDG_K11] + ([LDG_K12, LDG_K21] if second else []):
        r0, c0, v0 = ora.export_blocks(w)
        r1, c1, v1 = gpu.export_blocks(w)
        assert np.array_equal(r0, r1) and np.array_equal(c0, c1)
        assert rel(v1, v0) <= 1e-12
    x = case.normal_vector(gpu.m, 9)
    assert rel(gpu.spmv(LDG_K11, d(x)).cpu().numpy(), ora.spmv(LDG_K11, x)) <= 1e-12
    assert rel(gpu.split_matvec(0.2, d(x)).cpu().numpy(), ora.split_matvec(0.2, x)) <= 1e-12


@pytest.mark.gpu
def test_gpu_refused_inputs():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1204_1533_b200.linedg import ConfigError, LineDG

    empty = Case.custom(2, 2, np.zeros((0, 2)), np.zeros((0, 4), np.int32))
    with pytest.raises(ConfigError, match="no elements"):
        LineDG(empty, Physics(EU))
    big = Case.lattice(2, 1, 6)
    with pytest.raises(ConfigError, match="no sm_100a kernel"):
        LineDG(big, Physics(PO, bcs=[(t, [0.0]) for t in (1, 2, 3, 4)]))
