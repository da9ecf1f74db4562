"""Curved boundaries (reference mapping.cpp:30-65):
boundary-face nodes projected onto the true curve and the displacement
blended into the element (transfinite), pinned to the reference's OWN
compute_mapping with a CurveProjector, compiled unmodified from
/root/reference (oracle/ref_build), on an annulus around a cylinder (the
paper's geometry).  Known answers: projected nodes lie on
the circles, the quadrature area converges to pi (R1^2 - R0^2), free stream
is preserved on the curved mesh (the metric identities hold discretely).
"""
import ctypes as C
import math
import os

import numpy as np
import pytest

from paper_1204_1533_b200 import Case, _abi
from paper_1204_1533_b200._abi import dptr, host_lib
from paper_1204_1533_b200.cases import Physics, annulus_mesh

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libref_setup.so")
R0, R1 = 0.5, 3.0


def circle(x, y, tag):
    """Radial projection onto the circle of the face's tag (same formula and
    operation order as the setup library's built-in projector)."""
    r = R0 if tag == 1 else R1
    dx, dy = x - 0.0, y - 0.0
    s = r / math.sqrt(dx * dx + dy * dy)
    return 0.0 + s * dx, 0.0 + s * dy


def _ref():
    if not os.path.exists(REF_SO):
        if os.path.isdir("/root/reference/proj/src"):
            import subprocess

            subprocess.check_call([os.path.join(ROOT, "oracle", "ref_build", "build.sh")])
        else:
            pytest.skip("reference tree not present")
    L = C.CDLL(REF_SO)
    if not hasattr(L, "ref_case_remap"):
        pytest.skip("oracle/_ref predates the curved-mapping wrapper")
    vp, ip, dp = C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_double)
    L.ref_case_create.argtypes = [C.c_int, C.c_int, dp, C.c_int, ip, C.c_int, ip, C.c_int, ip, dp]
    L.ref_case_create.restype = vp
    L.ref_case_remap.argtypes = [vp, _abi.CURVE_FN, vp]
    L.ref_case_mapping.argtypes = [vp, dp, dp, dp, dp]
    L.ref_case_free.argtypes = [vp]
    L.ref_last_error.restype = C.c_char_p
    return L


def annulus(p, nr=3, nt=10, stretch=1.2):
    v, e, b = annulus_mesh(nr, nt, R0, R1, stretch)
    return v, e, b, Case.custom(2, p, v, e, b)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_curved_mapping_matches_reference(p):
    ref = _ref()
    v, e, b, case = annulus(p)
    case.remap(circle)
    h = ref.ref_case_create(p, len(v), dptr(np.ascontiguousarray(v)), len(e),
                            np.ascontiguousarray(e).ctypes.data_as(C.POINTER(C.c_int32)), len(b),
                            np.ascontiguousarray(b).ctypes.data_as(C.POINTER(C.c_int32)), 0, None, None)
    assert h, ref.ref_last_error()
    try:
        def _fn(_u, x, tag, out):
            out[0], out[1] = circle(x[0], x[1], tag)

        cb = _abi.CURVE_FN(_fn)
        assert ref.ref_case_remap(h, cb, None) == 0, ref.ref_last_error()
        npe, nq = (p + 1) ** 2, (3 * p + 2) // 2
        co, jac = np.zeros(case.E * npe * 2), np.zeros(case.E * npe)
        nv, ne = np.zeros(case.E * 2 * (p + 1) * nq * 2), np.zeros(case.E * 2 * 2 * (p + 1) * 2)
        ref.ref_case_mapping(h, dptr(co), dptr(jac), dptr(nv), dptr(ne))
        # node placement: same operations in the same order -> bitwise
        assert np.array_equal(co, case.coords.ravel())
        for a, b_ in ((jac, case.jac), (nv, case.nvec), (ne, case.normal_end)):
            b_ = b_.ravel()
            assert np.abs(a - b_).max() <= 1e-14 * np.abs(a).max()
    finally:
        ref.ref_case_free(h)


def test_builtin_circle_projector_equals_callback():
    _, _, _, a = annulus(4)
    _, _, _, b = annulus(4)
    a.remap(circle)
    b.remap_circles([(1, 0.0, 0.0, R0), (2, 0.0, 0.0, R1)])
    assert np.array_equal(a.coords, b.coords) and np.array_equal(a.jac, b.jac)
    assert np.array_equal(a.nvec, b.nvec) and np.array_equal(a.normal_end, b.normal_end)


def _area(case):
    n = case.np
    m = [np.zeros(k) for k in (n, case.nq, case.nq, n * case.nq, n * case.nq, n * n, n * n, n)]
    host_lib().lh_basis(case.p, 1, *[dptr(x) for x in m])
    w = np.multiply.outer(m[7], m[7]).T.reshape(-1)  # node i + n j
    return float((case.jac * w[None, :]).sum())


def test_projected_nodes_on_circles_and_area_converges():
    exact = math.pi * (R1 ** 2 - R0 ** 2)
    errs = []
    for p in (2, 3, 4):
        _, _, _, case = annulus(p, nr=2, nt=8, stretch=1.0)
        straight = abs(_area(case) - exact)
        case.remap_circles([(1, 0.0, 0.0, R0), (2, 0.0, 0.0, R1)])
        x = case.coords
        r = np.hypot(x[..., 0], x[..., 1])
        ef = case.elem_face()
        faces = case.faces()
        for el in range(case.E):
            for lf, sel in ((3, lambda k: k % (p + 1) == 0), (1, lambda k: k % (p + 1) == p)):
                f = faces[ef[el, lf]]
                if f[2] >= 0:
                    continue
                nodes = [k for k in range((p + 1) ** 2) if sel(k)]
                target = R0 if f[5] == 1 else R1
                assert np.abs(r[el, nodes] - target).max() < 1e-14 * target
        err = abs(_area(case) - exact)
        assert err < 0.02 * straight
        errs.append(err)
    assert errs[2] < errs[0]


@pytest.mark.parametrize("p", [2, 4])
def test_free_stream_preserved_on_curved_mesh(p):
    """SPEC acceptance 7 (p in {2, 4})."""
    from oracle.pyoracle import Oracle

    _, _, _, case = annulus(p)
    case.remap_circles([(1, 0.0, 0.0, R0), (2, 0.0, 0.0, R1)])
    g = 1.4
    st = [1.0, 0.5, 0.1, 1 / (g - 1) / g + 0.5 * (0.25 + 0.01)]
    U = np.tile(np.array(st), case.E * case.npe)
    for ri in (_abi.LDG_ROE, _abi.LDG_LLF):
        ph = Physics(_abi.LDG_EULER, riemann=ri, bcs=[(1, st), (2, st)])
        R = Oracle(case, ph).residual(U)
        assert np.abs(R).max() < 1e-11, np.abs(R).max()


def test_curved_3d_refused():
    case = Case.lattice(3, 2, 2)
    from paper_1204_1533_b200.linedg import ConfigError

    with pytest.raises(ConfigError):
        case.remap(lambda x, y, t: (x, y))
