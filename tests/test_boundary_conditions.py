"""Boundary conditions beyond Dirichlet: Neumann,
characteristic far field, slip wall, no-slip adiabatic wall (reference BcKind, physics.hpp:16-31;
PAPER.md:566-582), and curved boundaries
(mapping.cpp:30-65, tests/test_curved_mapping.py).

CPU: known answers and properties of the oracle restatement -- linear fields
are steady with exact Neumann data, slip walls conserve mass and energy
(zero normal mass flux through the mirrored-state Roe/LLF flux),
characteristic == Dirichlet against the far state, analytic Jacobians equal
finite differences (chain rule through the slip- and no-slip-wall ghost
states, the no-slip wall's component-dependent gradient trace), slip and
no-slip walls conserve mass and energy.  GPU (-m gpu): residual, gradient,
K11/K12/K21 patterns (bit-exact) and values, K11/K21 SpMV, split matvec and
the block-Jacobi preconditioner vs the oracle (<= 1e-12 / 1e-11).
"""
import numpy as np
import pytest

from paper_1204_1533_b200 import LDG_K11, LDG_K12, LDG_K21, Case, _abi
from paper_1204_1533_b200.cases import Physics, annulus_mesh

from oracle.pyoracle import Oracle

G = 1.4
EU, NS, PO = _abi.LDG_EULER, _abi.LDG_NAVIER_STOKES, _abi.LDG_POISSON
DIR, NEU, CHAR, SLIP, NOSLIP = (_abi.LDG_BC_DIRICHLET, _abi.LDG_BC_NEUMANN, _abi.LDG_BC_CHARACTERISTIC,
                                _abi.LDG_BC_SLIP_WALL, _abi.LDG_BC_NO_SLIP_ADIABATIC)


def rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    den = np.abs(b).max()
    return np.abs(a - b).max() / (den if den > 0 else 1.0)


def conservative(rho, vel, p):
    """(rho, rho u, E) per node from primitive arrays (D components of vel)."""
    D = len(vel)
    E = p / (G - 1) + 0.5 * rho * sum(v * v for v in vel)
    return np.stack([rho] + [rho * v for v in vel] + [E], axis=-1)


def flow_state(case, seed=0, amp=0.05, vel=None):
    """Smooth seeded perturbation of a uniform subsonic flow at the nodes."""
    rng = np.random.default_rng(seed)
    x = case.coords  # (E, npe, D)
    D = case.dim
    ph = rng.uniform(0, 2 * np.pi, size=(D + 2, D))
    waves = [sum(np.sin(1.3 * x[..., d] + ph[k, d]) for d in range(D)) for k in range(D + 2)]
    vel0 = vel if vel is not None else [0.3, -0.2, 0.1][:D]
    rho = 1.0 + amp * waves[0]
    v = [vel0[d] + amp * waves[1 + d] for d in range(D)]
    p = 1.0 / G + amp * waves[D + 1]
    return np.ascontiguousarray(conservative(rho, v, p).reshape(-1))


def box(dim, n, p, jitter=0.1, seed=3, rotate=True):
    return Case.lattice(dim, n, p, (1.0, 1.0, 1.0), jitter, False, False, True, rotate, seeds=(seed, seed + 1, seed + 2))


def node_weights(case):
    """Tensor GLL node weights x J (the quadrature of the residual's integral)."""
    n = case.np
    m = [np.zeros(k) for k in (n, case.nq, case.nq, n * case.nq, n * case.nq, n * n, n * n, n)]
    from paper_1204_1533_b200._abi import dptr, host_lib

    host_lib().lh_basis(case.p, 1, *[dptr(a) for a in m])
    w1 = m[7]
    w = w1
    for _ in range(case.dim - 1):
        w = np.multiply.outer(w, w1)
    # node index i + np*j (+ np^2 k): the last axis is i
    w = np.transpose(w, tuple(range(case.dim))[::-1]).reshape(-1)
    return w[None, :] * case.jac


# ------------------------------------------------------------ known answers
def test_linear_field_is_steady_with_neumann_data():
    """Poisson, u = a.x + b: with the exact Neumann flux g_N = -a.n on every
    side the LDG residual vanishes (linear fields are reproduced exactly)."""
    case = box(2, 4, 3)
    a = np.array([0.7, -0.4])
    x = case.coords
    U = np.ascontiguousarray((x @ a + 0.25).reshape(-1))
    normals = {1: (0, -1), 2: (1, 0), 3: (0, 1), 4: (-1, 0)}
    bcs = [(t, [-(a @ np.array(nv))], NEU) for t, nv in normals.items()]
    ora = Oracle(case, Physics(PO, bcs=bcs, c11_bd=1.0))
    R = ora.residual(U)
    assert np.abs(R).max() < 1e-10, np.abs(R).max()
    # the gradient is exact too (u_hat = u at Neumann boundaries)
    Q = ora.gradient(U).reshape(-1, 2)
    assert np.abs(Q - a).max() < 1e-11


def test_mixed_dirichlet_neumann_linear_field():
    """u = 2x on the unit square (boundary vertices are not jittered):
    Dirichlet g = 0 / 2 on the left / right sides, zero Neumann flux on the
    bottom / top -- the exact linear field is steady."""
    case = box(2, 3, 4, jitter=0.15)
    U = np.ascontiguousarray((2.0 * case.coords[..., 0]).reshape(-1))
    bcs = [(4, [0.0], DIR), (2, [2.0], DIR), (1, [0.0], NEU), (3, [0.0], NEU)]
    R = Oracle(case, Physics(PO, bcs=bcs)).residual(U)
    assert np.abs(R).max() < 1e-10, np.abs(R).max()


@pytest.mark.parametrize("riemann", [_abi.LDG_ROE, _abi.LDG_LLF])
@pytest.mark.parametrize("dim", [2, 3])
def test_slip_walls_conserve_mass_and_energy(riemann, dim):
    """A closed box with slip walls: the mirrored-state flux carries no mass
    or energy through the walls, so sum_nodes w J R_rho and R_E vanish."""
    case = box(dim, 3, 3 if dim == 2 else 2)
    U = flow_state(case, seed=5)
    bcs = [(t, [0.0] * (dim + 2), SLIP) for t in range(1, 2 * dim + 1)]
    ora = Oracle(case, Physics(EU, riemann=riemann, bcs=bcs))
    R = ora.residual(U).reshape(case.E, case.npe, dim + 2)
    w = node_weights(case)
    for comp in (0, dim + 1):
        tot = (w * R[..., comp]).sum()
        scale = (w * np.abs(R[..., comp])).sum()
        assert abs(tot) < 1e-12 * scale, (comp, tot, scale)
    # momentum is not conserved: the wall pressure acts on it
    assert abs((w * R[..., 1]).sum()) > 1e-8


def test_tangential_uniform_flow_along_slip_walls_is_steady():
    """Uniform flow parallel to straight slip walls (a channel, periodic in x)
    is an exact steady state."""
    n, p = 4, 3
    case = Case.lattice(2, n, p, (1.0, 1.0, 1.0), 0.0, False, False, False, False)
    v = case.vertices()
    el = case.elements()
    tl = case.tag_lines()
    ch = Case.custom(2, p, v, el, tl, periodic=[((4, 2), (1.0, 0.0))])
    U = np.tile(conservative(np.array(1.0), [np.array(0.4), np.array(0.0)], np.array(1 / G)),
                ch.E * ch.npe)
    bcs = [(1, [0] * 4, SLIP), (3, [0] * 4, SLIP)]
    for ri in (_abi.LDG_ROE, _abi.LDG_LLF):
        R = Oracle(ch, Physics(EU, riemann=ri, bcs=bcs)).residual(U)
        assert np.abs(R).max() < 1e-12


def test_characteristic_equals_dirichlet_far_state():
    case = box(2, 3, 3)
    U = flow_state(case, seed=2)
    far = list(conservative(np.array(1.0), [np.array(0.3), np.array(-0.2)], np.array(1 / G)))
    for kind in (EU, NS):
        mu = 1e-2 if kind == NS else 0.0
        a = Oracle(case, Physics(kind, mu=mu, bcs=[(t, far, CHAR) for t in (1, 2, 3, 4)]))
        b = Oracle(case, Physics(kind, mu=mu, bcs=[(t, far, DIR) for t in (1, 2, 3, 4)]))
        assert np.array_equal(a.residual(U), b.residual(U))


def _fd_check(case, phys, U, second):
    ora = Oracle(case, phys)
    ora.assemble(U)
    mats = [LDG_K11] + ([LDG_K12, LDG_K21] if second else [])
    Q = ora.gradient(U) if second else None
    for w in mats:
        A = ora.dense(w)
        F = ora.fd_dense(w, U, Q)
        assert rel(A, F) < 1e-6, (w, rel(A, F))
        # no finite-difference entry outside the analytic pattern
        rows, cols, _ = ora.export_blocks(w)
        br = A.shape[0] // (case.E * case.npe)
        bc = A.shape[1] // (case.E * case.npe)
        mask = np.zeros((case.E * case.npe, case.E * case.npe), dtype=bool)
        mask[rows, cols] = True
        big = np.abs(F).reshape(case.E * case.npe, br, case.E * case.npe, bc).max(axis=(1, 3))
        assert big[~mask].max(initial=0.0) < 1e-7 * np.abs(F).max()


@pytest.mark.parametrize("riemann", [_abi.LDG_ROE, _abi.LDG_LLF])
def test_euler_slip_characteristic_jacobian_vs_fd(riemann):
    verts, elems, btags = annulus_mesh(2, 8, 0.5, 2.0)
    case = Case.custom(2, 2, verts, elems, btags)
    case.remap_circles([(1, 0.0, 0.0, 0.5), (2, 0.0, 0.0, 2.0)])
    U = flow_state(case, seed=9)
    far = list(conservative(np.array(1.0), [np.array(0.3), np.array(0.0)], np.array(1 / G)))
    _fd_check(case, Physics(EU, riemann=riemann, bcs=[(1, [0] * 4, SLIP), (2, far, CHAR)]), U, False)


def test_navier_stokes_slip_neumann_jacobian_vs_fd():
    case = box(2, 2, 2)
    U = flow_state(case, seed=4)
    far = list(conservative(np.array(1.0), [np.array(0.3), np.array(-0.2)], np.array(1 / G)))
    bcs = [(1, [0] * 4, SLIP), (2, far, CHAR), (3, [0.0, 0.01, -0.02, 0.003], NEU), (4, far, DIR)]
    _fd_check(case, Physics(NS, mu=0.05, bcs=bcs), U, True)


def test_poisson_neumann_jacobian_vs_fd_and_pattern():
    case = box(2, 3, 3)
    U = np.ascontiguousarray(np.sin(3 * case.coords[..., 0]).reshape(-1))
    bcs = [(1, [0.3], NEU), (2, [0.0], DIR), (3, [-0.1], NEU), (4, [0.0], DIR)]
    _fd_check(case, Physics(PO, bcs=bcs), U, True)


def test_unsupported_boundary_kinds_are_refused():
    case = box(2, 2, 2)
    with pytest.raises(RuntimeError):
        Oracle(case, Physics(PO, bcs=[(t, [0.0], SLIP) for t in (1, 2, 3, 4)]))
    with pytest.raises(RuntimeError):
        Oracle(case, Physics(PO, bcs=[(t, [0.0], NOSLIP) for t in (1, 2, 3, 4)]))
    with pytest.raises(RuntimeError):
        Oracle(case, Physics(EU, bcs=[(t, [0.0] * 4, 7) for t in (1, 2, 3, 4)]))


@pytest.mark.parametrize("dim", [2, 3])
def test_no_slip_walls_conserve_mass_and_energy(dim):
    """A closed box of no-slip adiabatic walls: the reversed-
    momentum ghost carries no mass or energy through the wall, the adiabatic
    condition no viscous energy flux."""
    case = box(dim, 3, 3 if dim == 2 else 2)
    U = flow_state(case, seed=6)
    bcs = [(t, [0.0] * (dim + 2), NOSLIP) for t in range(1, 2 * dim + 1)]
    ora = Oracle(case, Physics(NS, mu=0.02, bcs=bcs))
    R = ora.residual(U).reshape(case.E, case.npe, dim + 2)
    w = node_weights(case)
    for comp in (0, dim + 1):
        tot = (w * R[..., comp]).sum()
        scale = (w * np.abs(R[..., comp])).sum()
        assert abs(tot) < 1e-12 * scale, (comp, tot, scale)
    # the gradient sees zero velocity at the wall: Q of momentum uses u_hat = 0
    Q = ora.gradient(U)
    assert np.isfinite(Q).all()


def test_no_slip_jacobians_vs_fd():
    """Mixed no-slip wall: component-dependent gradient trace (K21 rows of
    density and energy only) and the momentum penalty -- analytic = FD."""
    far = list(conservative(np.array(1.0), [np.array(0.3), np.array(-0.2)], np.array(1 / G)))
    case = box(2, 2, 2)
    U = flow_state(case, seed=4)
    bcs = [(1, [0] * 4, NOSLIP), (2, far, CHAR), (3, [0] * 4, NOSLIP), (4, far, DIR)]
    _fd_check(case, Physics(NS, mu=0.05, bcs=bcs), U, True)
    _fd_check(case, Physics(EU, bcs=bcs), U, False)
    case3 = box(3, 2, 1)
    U3 = flow_state(case3, seed=2)
    far3 = list(conservative(np.array(1.0), [np.array(0.2), np.array(0.1), np.array(-0.1)], np.array(1 / G)))
    bcs3 = [(1, far3, CHAR), (2, far3, CHAR), (3, [0] * 5, NOSLIP), (4, [0] * 5, NOSLIP), (5, [0] * 5, SLIP),
            (6, [0] * 5, NOSLIP)]
    _fd_check(case3, Physics(NS, mu=0.05, bcs=bcs3), U3, True)


# ------------------------------------------------------------- GPU parity
def _gpu_cases():
    """(name, builder) -> (case, physics, U, second_order)."""
    far2 = list(conservative(np.array(1.0), [np.array(0.3), np.array(0.05)], np.array(1 / G)))

    def cyl(p, riemann):
        def b():
            verts, elems, btags = annulus_mesh(3, 12, 0.5, 4.0, stretch=1.3)
            case = Case.custom(2, p, verts, elems, btags)
            case.remap_circles([(1, 0.0, 0.0, 0.5), (2, 0.0, 0.0, 4.0)])
            ph = Physics(EU, riemann=riemann, bcs=[(1, [0] * 4, SLIP), (2, far2, CHAR)])
            return case, ph, flow_state(case, seed=p), False
        return b

    def ns_box(p):
        def b():
            case = box(2, 3, p)
            bcs = [(1, [0] * 4, SLIP), (2, far2, CHAR), (3, [0.0, 0.01, -0.02, 0.003], NEU), (4, far2, DIR)]
            return case, Physics(NS, mu=0.02, bcs=bcs), flow_state(case, seed=11), True
        return b

    def poisson(p):
        def b():
            case = box(2, 4, p)
            bcs = [(1, [0.3], NEU), (2, [0.0], DIR), (3, [-0.1], NEU), (4, [0.5], DIR)]
            U = np.ascontiguousarray(np.sin(3 * case.coords[..., 0] + case.coords[..., 1]).reshape(-1))
            return case, Physics(PO, bcs=bcs), U, True
        return b

    def box3(kind, p, riemann=_abi.LDG_ROE):
        def b():
            case = box(3, 2, p, jitter=0.08)
            far3 = list(conservative(np.array(1.0), [np.array(0.2), np.array(0.1), np.array(-0.1)], np.array(1 / G)))
            bcs = [(1, far3, CHAR), (2, far3, CHAR), (3, [0] * 5, SLIP), (4, [0] * 5, SLIP),
                   (5, [0] * 5, SLIP), (6, [0.0, 0.0, 0.01, 0.0, 0.0], NEU)]
            mu = 0.02 if kind == NS else 0.0
            return case, Physics(kind, riemann=riemann, mu=mu, bcs=bcs), flow_state(case, seed=13), kind == NS
        return b

    def ns_noslip(p, dim=2):
        def b():
            case = box(dim, 3 if dim == 2 else 2, p)
            if dim == 2:
                bcs = [(1, [0] * 4, NOSLIP), (2, far2, CHAR), (3, [0] * 4, NOSLIP), (4, far2, DIR)]
            else:
                far3 = list(conservative(np.array(1.0), [np.array(0.2), np.array(0.1), np.array(-0.1)],
                                         np.array(1 / G)))
                bcs = [(1, far3, CHAR), (2, far3, CHAR), (3, [0] * 5, NOSLIP), (4, [0] * 5, NOSLIP),
                       (5, [0] * 5, SLIP), (6, [0] * 5, NOSLIP)]
            return case, Physics(NS, mu=0.02, bcs=bcs), flow_state(case, seed=17), True
        return b

    return [("ns-noslip-p3", ns_noslip(3)), ("ns-noslip-p4", ns_noslip(4)), ("ns3-noslip-p2", ns_noslip(2, 3)),
            ("cyl-p3-roe", cyl(3, _abi.LDG_ROE)), ("cyl-p4-roe", cyl(4, _abi.LDG_ROE)),
            ("cyl-p4-llf", cyl(4, _abi.LDG_LLF)), ("ns-box-p3", ns_box(3)), ("ns-box-p4", ns_box(4)),
            ("poisson-p3", poisson(3)), ("euler3-p3-llf", box3(EU, 3, _abi.LDG_LLF)),
            ("euler3-p2-roe", box3(EU, 2)), ("ns3-p2", box3(NS, 2)), ("ns3-p4", box3(NS, 4)),
            # 3-D p = 4 Euler: the line-streaming assembly with a whole direction per group
            ("euler3-p4-roe", box3(EU, 4)), ("euler3-p4-llf", box3(EU, 4, _abi.LDG_LLF))]


GPU = _gpu_cases()


@pytest.mark.gpu
@pytest.mark.parametrize("name,builder", GPU, ids=[g[0] for g in GPU])
def test_gpu_boundary_parity(name, builder):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1204_1533_b200.linedg import LineDG

    case, ph, U, second = builder()
    gpu = LineDG(case, ph)
    ora = Oracle(case, ph)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    host = lambda t: t.cpu().numpy()  # noqa: E731
    R0 = ora.residual(U)
    assert rel(host(gpu.residual(dev(U))), R0) <= 1e-12
    if second:
        assert rel(host(gpu.gradient_residual(dev(U))), ora.gradient(U)) <= 1e-12
    ora.assemble(U)
    gpu.assemble_jacobians(dev(U))
    for w in (LDG_K11, LDG_K12, LDG_K21) if second else (LDG_K11,):
        r0, c0, v0 = ora.export_blocks(w)
        r1, c1, v1 = gpu.export_blocks(w)
        assert np.array_equal(r0, r1) and np.array_equal(c0, c1), f"K{w} pattern"
        assert rel(v1, v0) <= 1e-12, (w, rel(v1, v0))
    x = case.normal_vector(gpu.m, 77)
    assert rel(host(gpu.spmv(LDG_K11, dev(x))), ora.spmv(LDG_K11, x)) <= 1e-12
    if second:
        assert rel(host(gpu.spmv(LDG_K21, dev(x))), ora.spmv(LDG_K21, x)) <= 1e-12
    for adt in (1e-3, 0.37):
        assert rel(host(gpu.split_matvec(adt, dev(x))), ora.split_matvec(adt, x)) <= 1e-12
    if case.dim == 2 and case.npe * gpu.m <= 128:
        # block-Jacobi preconditioner (K12 K21 on the element pattern, wall terms included)
        gpu.precond_build(0.05)
        ora.precond_build(0.05)
        assert rel(host(gpu.precond_apply(dev(x))), ora.precond_apply(x)) <= 1e-11


@pytest.mark.gpu
def test_gpu_refuses_poisson_walls():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1204_1533_b200.linedg import ConfigError, LineDG

    case = box(2, 2, 2)
    with pytest.raises(ConfigError, match="slip-wall"):
        LineDG(case, Physics(PO, bcs=[(t, [0.0], SLIP) for t in (1, 2, 3, 4)]))
    with pytest.raises(ConfigError, match="no-slip"):
        LineDG(case, Physics(PO, bcs=[(t, [0.0], NOSLIP) for t in (1, 2, 3, 4)]))
