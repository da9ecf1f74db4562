"""Block-Jacobi preconditioner + right-preconditioned GMRES (
SPEC.md:401-406, 429-447).

CPU part: the oracle against the SPEC known answers and a dense direct solve.
GPU part (`-m gpu`): the device preconditioner and GMRES against the oracle.
"""
import numpy as np
import pytest

from oracle.pyoracle import Oracle
from paper_1204_1533_b200 import CONFIGS, LDG_K11, LDG_K12, LDG_K21, Case, Physics, _abi

rng = np.random.default_rng(20261020)


def rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    den = np.abs(b).max()
    return np.abs(a - b).max() / (den if den > 0 else 1.0)


def ns_case(n=3, p=2):
    c = Case.lattice(2, n, p, jitter=0.1, periodic=True, permute=True, rotate=True, seeds=(11, 12, 13))
    ph = Physics(_abi.LDG_NAVIER_STOKES, mu=0.03)
    U = np.tile([1.0, 0.3, -0.2, 2.5], c.E * c.npe) + 0.02 * rng.standard_normal(c.E * c.npe * 4)
    return c, ph, U


def dense_system(o, adt, second):
    A = o.dense(LDG_K11)
    if second:
        A = A + o.dense(LDG_K12) @ o.dense(LDG_K21)
    return np.eye(A.shape[0]) - adt * A


def test_identity_operator_one_iteration():
    c, ph, U = ns_case()
    o = Oracle(c, ph)
    o.assemble(U)
    b = rng.standard_normal(o.n_dofs)
    x, it, conv, rn = o.gmres(0.0, b, rtol=1e-12, maxit=10, precond=False)
    assert conv and it == 1
    assert rel(x, b) <= 1e-14


def test_preconditioner_identity_at_zero_shift():
    c, ph, U = ns_case()
    o = Oracle(c, ph)
    o.assemble(U)
    o.precond_build(0.0)
    r = rng.standard_normal(o.n_dofs)
    assert np.array_equal(o.precond_apply(r), r)


def test_preconditioner_is_the_restricted_block_inverse():
    """z = (I - adt A~_e)^-1 r_e with A~ = A on the intra-element line pattern."""
    c, ph, U = ns_case()
    o = Oracle(c, ph)
    o.assemble(U)
    adt = 0.05
    M = dense_system(o, adt, True)
    n, ne = M.shape[0], c.npe * 4
    keep = np.zeros_like(M, dtype=bool)
    for e in range(c.E):
        for r in range(c.npe):
            for cc in range(c.npe):
                if (r % c.np == cc % c.np) or (r // c.np == cc // c.np):
                    keep[e * ne + r * 4:e * ne + r * 4 + 4, e * ne + cc * 4:e * ne + cc * 4 + 4] = True
    Mt = np.where(keep, M, 0.0)
    o.precond_build(adt)
    r = rng.standard_normal(n)
    z = o.precond_apply(r)
    assert rel(z, np.linalg.solve(Mt, r)) <= 1e-12


def test_gmres_matches_direct_solve():
    c, ph, U = ns_case()
    o = Oracle(c, ph)
    o.assemble(U)
    adt = 0.2
    M = dense_system(o, adt, True)
    b = rng.standard_normal(M.shape[0])
    xd = np.linalg.solve(M, b)
    for pc in (False, True):
        o.precond_build(adt)
        x, it, conv, rn = o.gmres(adt, b, rtol=1e-11, maxit=400, restart=60, precond=pc)
        assert conv, (pc, it, rn)
        assert np.linalg.norm(b - M @ x) <= 1e-10 * np.linalg.norm(b) * 1.01
        assert rel(x, xd) <= 1e-8
        assert abs(rn - np.linalg.norm(b - M @ x)) <= 1e-12 * np.linalg.norm(b)


def test_perfect_preconditioner_single_element():
    """One all-Dirichlet element, first-order physics: A~ = A (no fill, no neighbours),
    so preconditioned GMRES converges in one iteration."""
    c = Case.lattice(2, 1, 3, periodic=False)
    st = [1.0, 0.2, -0.1, 2.4]
    ph = Physics(_abi.LDG_EULER, bcs=[(t, st) for t in (1, 2, 3, 4)])
    U = np.tile(st, c.E * c.npe) + 0.01 * rng.standard_normal(c.E * c.npe * 4)
    o = Oracle(c, ph)
    o.assemble(U)
    adt = 0.3
    o.precond_build(adt)
    b = rng.standard_normal(o.n_dofs)
    x, it, conv, rn = o.gmres(adt, b, rtol=1e-10, maxit=5, precond=True)
    assert conv and it == 1
    assert rel(x, np.linalg.solve(dense_system(o, adt, False), b)) <= 1e-11


def test_block_jacobi_effectiveness_poisson_p3():
    """Poisson p=3, preconditioned GMRES needs >= 3x fewer iterations at rtol 1e-6.
    The ratio grows with the mesh (paper: ~20x at scale); on 16x16, adt=10 it is 3.1x
    (8x8: 2.1x), so the property is checked there."""
    cfg = CONFIGS[0]
    c, U = cfg.build(n=16)
    o = Oracle(c, cfg.physics)
    o.assemble(U)
    adt = 10.0
    o.precond_build(adt)
    b = rng.standard_normal(o.n_dofs)
    _, it_pc, conv_pc, _ = o.gmres(adt, b, rtol=1e-6, maxit=3000, restart=300, precond=True)
    _, it_no, conv_no, _ = o.gmres(adt, b, rtol=1e-6, maxit=3000, restart=300, precond=False)
    assert conv_pc and conv_no
    assert it_no >= 3 * it_pc, (it_no, it_pc)


# ---------------------------------------------------------------- GPU parity
def test_precond_inverse_mode_equals_lu():
    """ldg_set_precond_mode(1): explicit block inverses -- the same operator as
    the LU solves to round-off."""
    cfg = CONFIGS[2]
    c, U = cfg.build(n=3)
    o = Oracle(c, cfg.physics)
    o.assemble(U)
    r = rng.standard_normal(o.n_dofs)
    o.precond_build(0.05)
    z_lu = o.precond_apply(r)
    o.set_precond_mode(1)
    o.precond_build(0.05)
    z_inv = o.precond_apply(r)
    assert rel(z_inv, z_lu) <= 1e-12


def test_line_adi_preconditioner_3d():
    """3-D p >= 2 (element blocks above 128 unknowns): the line-ADI
    preconditioner -- exact on a single line (1-D
    coupling only: it is then the block inverse), and it cuts GMRES
    iterations on the 3-D Navier-Stokes and Euler configurations."""
    for ci, n, adt, gain in ((4, 3, 0.05, 0.8), (3, 2, 0.05, 0.9)):
        cfg = CONFIGS[ci]
        c, U = cfg.build(n=n)
        o = Oracle(c, cfg.physics)
        o.assemble(U)
        o.precond_build(adt)
        b = c.normal_vector(o.m, cfg.vector_seed)
        _, it_pc, cv_pc, _ = o.gmres(adt, b, rtol=1e-8, maxit=300, restart=60, precond=True)
        _, it_no, cv_no, _ = o.gmres(adt, b, rtol=1e-8, maxit=300, restart=60, precond=False)
        assert cv_pc and cv_no and it_pc < gain * it_no, (ci, it_pc, it_no)
    # mode 2 forces line-ADI on a 2-D configuration as well; at alpha_dt = 0 it is the identity
    cfg = CONFIGS[1]
    c, U = cfg.build(n=3)
    o = Oracle(c, cfg.physics)
    o.assemble(U)
    o.set_precond_mode(2)
    o.precond_build(0.0)
    r = c.normal_vector(o.m, 77)
    assert np.array_equal(o.precond_apply(r), r)
    with pytest.raises(Exception):
        o.set_precond_mode(3)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1, 2], ids=["auto", "inverse", "line-adi"])
@pytest.mark.parametrize("ci,n", [(0, 4), (1, 4), (2, 3), (3, 2), (4, 2)])
def test_gpu_preconditioner_and_gmres(ci, n, mode):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1204_1533_b200.linedg import LineDG

    cfg = CONFIGS[ci]
    if mode == 1 and ci >= 3:
        pytest.skip("element inverses: element blocks of up to 128 unknowns")
    c, U = cfg.build(n=n)
    o = Oracle(c, cfg.physics)
    g = LineDG(c, cfg.physics)
    o.set_precond_mode(mode)
    g.set_precond_mode(mode)
    src = cfg.source_for(c)
    if src is not None:
        o.set_source(src)
        g.set_source(src)
    o.assemble(U)
    g.assemble_jacobians(U)
    for adt in (0.0, 0.05, 1.0):
        o.precond_build(adt)
        g.precond_build(adt)
        r = rng.standard_normal(o.n_dofs)
        assert rel(g.precond_apply(r), o.precond_apply(r)) <= 1e-11, adt
    adt = 0.05
    o.precond_build(adt)
    g.precond_build(adt)
    b = rng.standard_normal(o.n_dofs)
    for pc in (True, False):
        # a fixed number of iterations (no early exit): same Krylov space
        x0, it0, _, r0 = o.gmres(adt, b, rtol=1e-30, maxit=8, restart=8, precond=pc)
        x1, it1, _, r1 = g.gmres(adt, b, rtol=1e-30, maxit=8, restart=8, precond=pc)
        assert it0 == it1 == 8
        assert rel(x1, x0) <= 1e-9, (pc, rel(x1, x0))
        assert abs(r1 - r0) <= 1e-9 * np.linalg.norm(b)
        # converged solve
        x0, it0, cv0, _ = o.gmres(adt, b, rtol=1e-9, maxit=300, restart=50, precond=pc)
        x1, it1, cv1, _ = g.gmres(adt, b, rtol=1e-9, maxit=300, restart=50, precond=pc)
        if mode == 2 and pc and not cv0:
            # line-ADI on a stiff 2-D operator (Poisson, alpha_dt = 0.05): the
            # O(alpha_dt^2) splitting error can stall GMRES -- both sides alike
            assert not cv1
            continue
        assert cv0 and cv1 and abs(it0 - it1) <= 1
        assert rel(x1, x0) <= 1e-7


@pytest.mark.gpu
@pytest.mark.slow
def test_gpu_line_adi_full_size():
    """Full-size C4 (3-D Euler p = 3, 64^3, 84 M DOFs): the line-ADI factors
    (40 GB next to the 54 GB Jacobian) build on one B200 and cut the GMRES
    iterations; C5 (164 GB Jacobian) has no room for its 41 GB of factors and
    reports it as a configuration error instead of failing an allocation."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1204_1533_b200.linedg import ConfigError, LineDG

    cfg = CONFIGS[3]
    c, U = cfg.build()
    g = LineDG(c, cfg.physics)
    Ud = torch.from_numpy(U).cuda()
    g.assemble_jacobians(Ud)
    adt = 0.002
    import time
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g.precond_build(adt)
    t_build = time.perf_counter() - t0
    b = torch.from_numpy(c.normal_vector(g.m, cfg.vector_seed)).cuda()
    bn = float(torch.linalg.norm(b))
    # 20 iterations each (no early exit): the preconditioned residual is smaller
    _, _, _, r_pc = g.gmres(adt, b, rtol=1e-30, maxit=20, restart=20, precond=True)
    _, _, _, r_no = g.gmres(adt, b, rtol=1e-30, maxit=20, restart=20, precond=False)
    print(f"C4 full line-ADI: build {t_build:.2f} s; ||b - Ax|| / ||b|| after 20 GMRES iterations "
          f"{r_pc / bn:.3e} (unpreconditioned {r_no / bn:.3e})")
    assert r_pc < r_no
    g.close()
    del Ud, b
    cfg = CONFIGS[4]
    c, U = cfg.build()
    g = LineDG(c, cfg.physics)
    g.assemble_jacobians(torch.from_numpy(U).cuda())
    with pytest.raises(ConfigError, match="free"):
        g.precond_build(0.002)
    g.close()
