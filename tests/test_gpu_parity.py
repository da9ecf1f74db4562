"""GPU (sm_100a) vs CPU oracle parity through the C-ABI.

Bar (BASELINE.json north_star): residuals, gradients and Jacobian values to a
normwise relative L-infinity error <= 1e-12 (err = max|a-b| / max|b|,
SURVEY.md Appendix B), node sparsity patterns and indexing bit-exact.
"""
import numpy as np
import pytest

from paper_1204_1533_b200 import CONFIGS, LDG_K11, LDG_K12, LDG_K21, Case, Physics, _abi
from paper_1204_1533_b200.linedg import ConfigError, LineDG, PhysicalStateError

pytestmark = pytest.mark.gpu

TOL = 1e-12

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - GPU marker tests only run on the box
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle.pyoracle import Oracle  # noqa: E402  (test infrastructure)


def rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    den = np.abs(b).max()
    return np.abs(a - b).max() / (den if den > 0 else 1.0)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


# (config index, n, rotate override)
SMALL = [(0, 4, None), (0, 4, False), (1, 4, None), (1, 4, True), (2, 4, None), (2, 4, True),
         (3, 2, None), (3, 3, False), (4, 2, None), (4, 2, True)]


def small_ids():
    return [f"C{c + 1}-n{n}-rot{r}" for c, n, r in SMALL]


@pytest.fixture(scope="module", params=SMALL, ids=small_ids())
def setup(request):
    ci, n, rot = request.param
    cfg = CONFIGS[ci]
    case, U = cfg.build(n=n, rotate=rot)
    src = cfg.source_for(case)
    gpu = LineDG(case, cfg.physics)
    ora = Oracle(case, cfg.physics)
    if src is not None:
        gpu.set_source(src)
        ora.set_source(src)
    return cfg, case, U, gpu, ora


def test_residual(setup):
    cfg, case, U, gpu, ora = setup
    R_ref = ora.residual(U)
    R = host(gpu.residual(dev(U)))
    assert rel(R, R_ref) <= TOL, rel(R, R_ref)


def test_residual_host_path(setup):
    cfg, case, U, gpu, ora = setup
    R_ref = ora.residual(U)
    R = gpu.residual(U)  # numpy in -> host path through the C-ABI
    assert rel(R, R_ref) <= TOL
    # into a caller-provided pinned buffer (bench.py's end-to-end leg)
    Rp = torch.empty(R.size, dtype=torch.float64).pin_memory().numpy()
    assert gpu.residual(U, out=Rp) is Rp
    assert np.array_equal(Rp, R)
    # host-path Jacobian + SpMV / split matvec into pinned buffers
    gpu.assemble_jacobians(U)
    ora.assemble(U)
    x = case.normal_vector(gpu.m, cfg.vector_seed)
    yp = torch.empty(x.size, dtype=torch.float64).pin_memory().numpy()
    assert gpu.spmv(LDG_K11, x, out=yp) is yp
    assert rel(yp, ora.spmv(LDG_K11, x)) <= TOL
    assert rel(gpu.split_matvec(0.37, x, out=yp), ora.split_matvec(0.37, x)) <= TOL
    with pytest.raises(ValueError):
        gpu.residual(U, out=np.empty(3))


def test_gradient_and_second_order(setup):
    cfg, case, U, gpu, ora = setup
    if not cfg.physics.second_order():
        pytest.skip("first-order physics")
    Q_ref = ora.gradient(U)
    Q = host(gpu.gradient_residual(dev(U)))
    assert rel(Q, Q_ref) <= TOL
    # R(U, Q) at an independent Q exercises the K12 path of the residual
    rng = np.random.default_rng(7)
    Qr = Q_ref + 0.1 * np.abs(Q_ref).max() * rng.standard_normal(Q_ref.shape)
    R_ref = ora.residual_uq(U, Qr)
    R = host(gpu.residual_second_order(dev(U), dev(Qr)))
    assert rel(R, R_ref) <= TOL


def _matrices(cfg):
    return (LDG_K11, LDG_K12, LDG_K21) if cfg.physics.second_order() else (LDG_K11,)


def test_jacobian_pattern_and_values(setup):
    cfg, case, U, gpu, ora = setup
    ora.assemble(U)
    gpu.assemble_jacobians(dev(U))
    for w in _matrices(cfg):
        r0, c0, v0 = ora.export_blocks(w)
        r1, c1, v1 = gpu.export_blocks(w)
        assert np.array_equal(r0, r1), f"K{w} rows differ"
        assert np.array_equal(c0, c1), f"K{w} cols differ"
        assert v1.shape == v0.shape
        assert rel(v1, v0) <= TOL, (w, rel(v1, v0))
        info = gpu.pattern_info(w)
        assert info.nnzb == len(r0)


def test_spmv_and_split(setup):
    cfg, case, U, gpu, ora = setup
    ora.assemble(U)
    gpu.assemble_jacobians(dev(U))
    m = gpu.m
    x = case.normal_vector(m, cfg.vector_seed)
    y_ref = ora.spmv(LDG_K11, x)
    y = host(gpu.spmv(LDG_K11, dev(x)))
    assert rel(y, y_ref) <= TOL
    if cfg.physics.second_order():
        w_ref = ora.spmv(LDG_K21, x)
        w = host(gpu.spmv(LDG_K21, dev(x)))
        assert rel(w, w_ref) <= TOL
        z_ref = ora.spmv(LDG_K12, w_ref)
        z = host(gpu.spmv(LDG_K12, dev(w_ref)))
        assert rel(z, z_ref) <= TOL
    for adt in (0.0, 1e-3, 0.37):
        s_ref = ora.split_matvec(adt, x)
        s = host(gpu.split_matvec(adt, dev(x)))
        assert rel(s, s_ref) <= TOL
    # alpha_dt = 0 returns v bitwise
    assert np.array_equal(host(gpu.split_matvec(0.0, dev(x))), x)


def test_physical_state_error():
    cfg = CONFIGS[1]
    case, U = cfg.build(n=4)
    gpu = LineDG(case, cfg.physics)
    U = U.copy()
    U[4 * 37] = -1.0  # negative density at node 37
    with pytest.raises(PhysicalStateError) as ei:
        gpu.residual(dev(U))
    st = ei.value.state
    rho, mom, E = st[0], st[1:3], st[3]
    p = 0.4 * (E - 0.5 * (mom @ mom) / rho) if rho != 0 else -1
    assert rho <= 0 or p <= 0


def test_missing_boundary_condition_is_config_error():
    case = Case.lattice(2, 3, 2)
    with pytest.raises(ConfigError):
        LineDG(case, Physics(_abi.LDG_EULER))


@pytest.mark.slow
def test_full_c2_residual_and_jacobian_rows():
    cfg = CONFIGS[1]
    case, U = cfg.build()
    gpu = LineDG(case, cfg.physics)
    ora = Oracle(case, cfg.physics)
    R_ref = ora.residual(U)
    R = host(gpu.residual(dev(U)))
    assert rel(R, R_ref) <= TOL
    rng = np.random.default_rng(3)
    elems = np.sort(rng.choice(case.E, 64, replace=False)).astype(np.int32)
    ora.assemble(U, elems=elems)
    gpu.assemble_jacobians(dev(U))
    r0, c0, v0 = ora.export_blocks(LDG_K11)
    keep = np.isin(r0 // case.npe, elems)
    r1, c1, v1 = gpu.export_blocks(LDG_K11, elems=elems)
    assert np.array_equal(r0[keep], r1) and np.array_equal(c0[keep], c1)
    assert rel(v1, v0[keep]) <= TOL
    # Table 1 on the full config mesh: 2p+5 node columns per K11 row (periodic)
    info = gpu.pattern_info(LDG_K11)
    assert info.nnzb == (2 * cfg.p + 5) * case.E * case.npe


@pytest.mark.parametrize("ci", [1, 2], ids=["C2-n96", "C3-n96"])
def test_large_mesh_assembly_rows_match_oracle(ci):
    """A 9216-element mesh (persistent assembly with many elements per CTA):
    K11 (+ K12, K21) rows of 64 random elements against the oracle, and a
    repeated assembly reproduces them bitwise."""
    cfg = CONFIGS[ci]
    case, U = cfg.build(n=96)
    gpu = LineDG(case, cfg.physics)
    ora = Oracle(case, cfg.physics)
    rng = np.random.default_rng(5)
    elems = np.sort(rng.choice(case.E, 64, replace=False)).astype(np.int32)
    ora.assemble(U, elems=elems)
    gpu.assemble_jacobians(dev(U))
    first = None
    for w in _matrices(cfg):
        r0, c0, v0 = ora.export_blocks(w)
        keep = np.isin(r0 // case.npe, elems)
        r1, c1, v1 = gpu.export_blocks(w, elems=elems)
        assert np.array_equal(r0[keep], r1) and np.array_equal(c0[keep], c1)
        assert rel(v1, v0[keep]) <= TOL, (w, rel(v1, v0[keep]))
        if first is None:
            first = v1
    gpu.assemble_jacobians(dev(U))
    assert np.array_equal(gpu.export_blocks(LDG_K11, elems=elems)[2], first)


def test_async_host_path_matches_sync():
    """ldg_set_sync_errors(ctx, 0): host-buffer calls run on the copy streams
    and return early; after synchronize() the results equal the synchronous
    ones bitwise (C2 scaled and C3 scaled: second-order Q download too)."""
    for ci in (1, 2):
        cfg = CONFIGS[ci]
        case, U = cfg.build(n=8)
        gpu = LineDG(case, cfg.physics)
        x = case.normal_vector(gpu.m, cfg.vector_seed)
        R0 = gpu.residual(U)
        gpu.assemble_jacobians(U)
        y0 = gpu.spmv(LDG_K11, x)
        Rp = torch.empty(R0.size, dtype=torch.float64).pin_memory().numpy()
        yp = torch.empty(y0.size, dtype=torch.float64).pin_memory().numpy()
        Up = torch.from_numpy(U).pin_memory().numpy()
        xp = torch.from_numpy(x).pin_memory().numpy()
        gpu.set_sync_errors(False)
        for _ in range(3):  # repeated calls reuse the staging buffers (event-ordered)
            Rp[:] = 0.0
            yp[:] = 0.0
            gpu.residual(Up, out=Rp)
            gpu.assemble_jacobians(Up)
            gpu.spmv(LDG_K11, xp, out=yp)
            gpu.synchronize()
            assert np.array_equal(Rp, R0) and np.array_equal(yp, y0)
        gpu.set_sync_errors(True)
        # synchronous call into pinned memory: the zero-copy product (M = 4)
        yp[:] = 0.0
        gpu.spmv(LDG_K11, xp, out=yp)
        assert np.array_equal(yp, y0)
        ora = Oracle(case, cfg.physics)
        ora.assemble(U)
        assert rel(y0, ora.spmv(LDG_K11, x)) <= TOL


def _with_neighbours(ora, case, elems):
    """elems plus the elements their K12 (switch-side) columns reach: the K21
    rows a split matvec over the rows of `elems` consumes."""
    r, c, _ = ora.export_blocks(LDG_K12)
    keep = np.isin(r // case.npe, elems)
    return np.unique(np.concatenate([elems, (c[keep] // case.npe).astype(np.int32)])).astype(np.int32)


@pytest.mark.slow
@pytest.mark.parametrize("ci", [2, 3, 4], ids=["C3-full", "C4-full", "C5-full"])
def test_full_size_rows_match_oracle(ci):
    """Full BASELINE.json sizes (C3 6.6 M, C4 84 M, C5 69 M DOFs; C5's store is
    164 GB) on the configs' OWN states (no perturbation): on the DOFs of 32
    random elements, the residual, the K11 (+ K12, K21) rows, the K11 product
    and the split matvec against the oracle evaluated on those elements only,
    and the Table-1 node-column counts of the whole K11 pattern.

    Residual tolerance.  C3 and C5 are near-steady: their residual is a 1e4-fold
    cancellation of O(p^2/h) line terms, so ANY fp64 evaluation carries a
    normwise error far above 1e-12 -- the oracle itself moves by 3e-10 (C3) /
    4e-11 (C5) between an FMA-contracted and an uncontracted build, and lies
    2e-10 / 6e-11 from the same restatement evaluated in long double
    (DESIGN.md section 3).  The bar on the own state is therefore accuracy:
    the GPU residual must sit on the same fp64 conditioning floor as the
    oracle -- within twice the oracle's own distance from the extended-
    precision evaluation (or within 1e-12 of it).  The 1e-12
    GPU-vs-oracle bar itself is checked on a seeded 2 % perturbation of the
    same state (an O(n) residual on the same code paths)."""
    cfg = CONFIGS[ci]
    case, U = cfg.build()
    gpu = LineDG(case, cfg.physics)
    try:
        ora = Oracle(case, cfg.physics)
        rng = np.random.default_rng(11)
        elems = np.sort(rng.choice(case.E, 32, replace=False)).astype(np.int32)
        m = gpu.m
        dofs = (elems[:, None] * case.npe * m + np.arange(case.npe * m)[None, :]).ravel()
        # residual on the config's own state: accuracy against long double
        R = host(gpu.residual(dev(U)))[dofs]
        R64 = ora.residual(U, elems=elems)[dofs]
        Rx = ora.residual_ext(U, elems=elems)[dofs]
        e_gpu, e_ora = rel(R, Rx), rel(R64, Rx)
        print(f"C{ci + 1} residual: gpu-vs-ext {e_gpu:.3e}  oracle64-vs-ext {e_ora:.3e}  "
              f"gpu-vs-oracle64 {rel(R, R64):.3e}")
        assert e_gpu <= max(TOL, 2.0 * e_ora), (e_gpu, e_ora)
        # the 1e-12 bar against the fp64 oracle on an O(n) residual
        Up = U * (1.0 + 0.02 * np.random.default_rng(12).standard_normal(U.shape))
        Rp = host(gpu.residual(dev(Up)))
        assert rel(Rp[dofs], ora.residual(Up, elems=elems)[dofs]) <= TOL
        del Rp, Up
        # Jacobian rows, K11 product and split matvec on the config's own state
        gpu.assemble_jacobians(dev(U))
        ora.assemble(U, elems=elems)
        for w in _matrices(cfg):
            r0, c0, v0 = ora.export_blocks(w)
            keep = np.isin(r0 // case.npe, elems)
            r1, c1, v1 = gpu.export_blocks(w, elems=elems)
            assert np.array_equal(r0[keep], r1) and np.array_equal(c0[keep], c1), f"K{w} pattern"
            assert rel(v1, v0[keep]) <= TOL, (w, rel(v1, v0[keep]))
        per_row = 2 * cfg.p + 5 if case.dim == 2 else 3 * cfg.p + 7
        assert gpu.pattern_info(LDG_K11).nnzb == per_row * case.E * case.npe
        x = case.normal_vector(m, cfg.vector_seed)
        xd = dev(x)
        y = host(gpu.spmv(LDG_K11, xd))[dofs]
        assert rel(y, ora.spmv(LDG_K11, x)[dofs]) <= TOL
        if cfg.physics.second_order():  # K21 rows of the neighbours the K12 columns reach
            ora.assemble(U, elems=_with_neighbours(ora, case, elems))
        for adt in (1e-3, 0.37):
            s = host(gpu.split_matvec(adt, xd))[dofs]
            assert rel(s, ora.split_matvec(adt, x)[dofs]) <= TOL, adt
    finally:
        gpu.close()


@pytest.mark.parametrize("ci", [1, 2, 3, 4], ids=["C2", "C3", "C4", "C5"])
def test_spmv_row_orders(ci):
    """Both row walks of the block SpMV / split matvec (LDG_OPT_SPMV_ROW_ORDER:
    forward, taken by every store above 1 GiB -- C3, C4, C5 at full size -- and
    reverse, taken by small stores) against the oracle, and bitwise equal to
    each other."""
    cfg = CONFIGS[ci]
    case, U = cfg.build(n=4 if cfg.dim == 2 else 3)
    gpu = LineDG(case, cfg.physics)
    ora = Oracle(case, cfg.physics)
    ora.assemble(U)
    gpu.assemble_jacobians(dev(U))
    x = case.normal_vector(gpu.m, cfg.vector_seed)
    y_ref = ora.spmv(LDG_K11, x)
    s_ref = ora.split_matvec(0.37, x)
    out = []
    for order in (1, 2):
        gpu.set_option(_abi.LDG_OPT_SPMV_ROW_ORDER, order)
        y = host(gpu.spmv(LDG_K11, dev(x)))
        s = host(gpu.split_matvec(0.37, dev(x)))
        assert rel(y, y_ref) <= TOL and rel(s, s_ref) <= TOL, order
        out.append((y, s))
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
    with pytest.raises(Exception):
        gpu.set_option(_abi.LDG_OPT_SPMV_ROW_ORDER, 3)


def test_two_contexts_concurrent_threads():
    """Two contexts of different configurations (2-D Euler, 2-D Navier-Stokes)
    driven from two host threads at once: per-device launch state is shared
    and thread-safe, results equal the single-threaded ones bitwise and the
    oracle to 1e-12."""
    import threading

    cases = []
    for ci in (1, 2):
        cfg = CONFIGS[ci]
        case, U = cfg.build(n=6)
        cases.append((cfg, case, U, case.normal_vector(cfg.physics.components(case.dim), cfg.vector_seed)))

    def run(cfg, case, U, x, out):
        g = LineDG(case, cfg.physics)
        for _ in range(3):
            R = g.residual(U)
            g.assemble_jacobians(U)
            y = g.split_matvec(0.37, x)
        out.append((R, y))
        g.close()

    ref = []
    for c in cases:
        o = []
        run(*c, o)
        ref.append(o[0])
    outs = [[], []]
    th = [threading.Thread(target=run, args=(*cases[i], outs[i])) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for i, (cfg, case, U, x) in enumerate(cases):
        assert np.array_equal(outs[i][0][0], ref[i][0]) and np.array_equal(outs[i][0][1], ref[i][1])
        ora = Oracle(case, cfg.physics)
        assert rel(ref[i][0], ora.residual(U)) <= TOL
        ora.assemble(U)
        assert rel(ref[i][1], ora.split_matvec(0.37, x)) <= TOL
