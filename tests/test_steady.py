"""Pseudo-transient continuation to a steady state (
SPEC.md:515-536; "a sequence of increasing timesteps and a
final step without the time derivatives", backward Euler).

CPU (oracle restatement lo_steady_solve): the SPEC known answers -- a steady
U0 returns after one residual check; Poisson (linear) converges in exactly one
final-phase Newton update whatever the schedule; the inviscid cylinder
(slip wall + characteristic far field, curved annulus) started from free
stream reaches ||R||_inf < 1e-10; runs are deterministic.  GPU (-m gpu): the
device driver ldg_steady_solve mirrors the oracle -- identical counts and
states within 1e-9 for the linear problem, the same steady state (1e-8) within
one update for the cylinder, and the per-update CSV log.
"""
import numpy as np
import pytest

from paper_1204_1533_b200 import CONFIGS, Case, _abi
from paper_1204_1533_b200.cases import Physics, annulus_mesh

from oracle.pyoracle import Oracle

G = 1.4
M_INF = 0.3
FAR = [1.0, M_INF, 0.0, 1 / (G * (G - 1)) + 0.5 * M_INF * M_INF]


def cylinder(p=2, nr=4, nt=16):
    v, e, b = annulus_mesh(nr, nt, 0.5, 6.0, stretch=1.4)
    case = Case.custom(2, p, v, e, b)
    case.remap_circles([(1, 0.0, 0.0, 0.5), (2, 0.0, 0.0, 6.0)])
    ph = Physics(_abi.LDG_EULER, bcs=[(1, [0] * 4, _abi.LDG_BC_SLIP_WALL), (2, FAR, _abi.LDG_BC_CHARACTERISTIC)])
    return case, ph, np.tile(np.array(FAR), case.E * case.npe)


def cyl_cfg(**kw):
    base = dict(dt0=0.01, growth=1.3, n_steps=30, gmres_iters=60, gmres_rtol=1e-3, newton_tol=1e-10, max_newton=20)
    base.update(kw)
    return _abi.steady_cfg(**base)


def poisson(n=8):
    cfg = CONFIGS[0]
    case, U = cfg.build(n=n)
    return case, cfg.physics, U, cfg.source_for(case)


def test_steady_initial_state_returns_after_one_residual():
    cfg = CONFIGS[1]
    case, _ = cfg.build(n=4)
    U = np.tile(np.array([1.0, 0.5, 0.2, 2.5]), case.E * case.npe)  # free stream, periodic
    ora = Oracle(case, cfg.physics)
    Us, st = ora.steady_solve(U, _abi.steady_cfg(newton_tol=1e-10))
    assert np.array_equal(Us, U)
    assert st["residual_evals"] == 1 and st["newton_iters"] == 0 and st["jacobian_assemblies"] == 0


@pytest.mark.parametrize("dt0,growth,n_steps", [(1e-3, 2.0, 3), (0.1, 1.5, 6), (1e-2, 2.0, 0)])
def test_poisson_converges_in_one_final_newton_update(dt0, growth, n_steps):
    case, ph, U, src = poisson()
    ora = Oracle(case, ph)
    ora.set_source(src)
    sc = _abi.steady_cfg(dt0=dt0, growth=growth, n_steps=n_steps, gmres_iters=400, gmres_rtol=1e-13,
                         newton_tol=1e-9, max_newton=3)
    Us, st = ora.steady_solve(U, sc)
    assert st["newton_iters"] == n_steps + 1, st
    assert np.abs(ora.residual(Us)).max() <= 1e-9


def test_cylinder_from_free_stream_reaches_steady_state():
    case, ph, U0 = cylinder()
    ora = Oracle(case, ph)
    Us, st = ora.steady_solve(U0, cyl_cfg())
    assert st["residual_norm"] < 1e-10 and st["newton_iters"] <= 40, st
    assert np.abs(ora.residual(Us)).max() < 1e-10
    # the slip wall turns the flow: the steady state is not the free stream
    assert np.abs(Us - U0).max() > 1e-2
    # deterministic (fixed-order reductions)
    Us2, st2 = ora.steady_solve(U0, cyl_cfg())
    assert st2 == st and np.array_equal(Us, Us2)


def test_hopeless_schedule_reports_divergence():
    case, ph, U0 = cylinder(nr=3, nt=12)
    ora = Oracle(case, ph)
    with pytest.raises(RuntimeError, match="diverged|converge"):
        ora.steady_solve(U0, cyl_cfg(dt0=5.0, growth=4.0, n_steps=2, max_newton=2, gmres_iters=5))


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["poisson", "cylinder"])
def test_gpu_steady_solve_matches_oracle(which, tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1204_1533_b200.linedg import LineDG

    if which == "poisson":
        case, ph, U0, src = poisson()
        sc = dict(dt0=1e-3, growth=2.0, n_steps=3, gmres_iters=120, gmres_rtol=0.0, newton_tol=1e-9, max_newton=4)
    else:
        case, ph, U0 = cylinder(nr=3, nt=12)
        src = None
        sc = dict(dt0=0.01, growth=1.3, n_steps=30, gmres_iters=40, gmres_rtol=0.0, newton_tol=1e-10, max_newton=20)
    gpu = LineDG(case, ph)
    ora = Oracle(case, ph)
    if src is not None:
        gpu.set_source(src)
        ora.set_source(src)
    U1, s1 = ora.steady_solve(U0, _abi.steady_cfg(**sc))
    log = tmp_path / "steady.csv"
    U2, s2 = gpu.steady_solve(U0, _abi.steady_cfg(log_csv=str(log), **sc))
    if which == "poisson":
        # linear problem: the same updates, counts and state to round-off
        for k in ("newton_iters", "gmres_iters", "jacobian_assemblies", "residual_evals"):
            assert s1[k] == s2[k], (k, s1, s2)
        assert np.abs(U2 - U1).max() <= 1e-9 * np.abs(U1).max()
    else:
        # nonlinear continuation with fixed-length GMRES: round-off moves the
        # path by a few updates; both end at the same steady state
        assert abs(s1["newton_iters"] - s2["newton_iters"]) <= 3, (s1, s2)
        assert s2["residual_norm"] <= 1e-10
        assert np.abs(U2 - U1).max() <= 1e-8 * np.abs(U1).max()
    rows = log.read_text().splitlines()
    assert rows[0] == "step,stage,newton_iters,gmres_iters,jacobian_refreshed,residual_norm"
    body = [r.split(",") for r in rows[1:]]
    assert len(body) == s2["newton_iters"]
    assert float(body[-1][5]) == pytest.approx(s2["residual_norm"], rel=0, abs=0)
    assert body[-1][1] == "1"  # converged in the final (Newton) phase
