"""Wire formats: the reference mesh text file
(load_mesh / save_mesh, mesh.cpp:115-166), the matrix triplet export
`i j value` and the sparsity-summary CSV `p,avg_cols_per_block_row,nnz`
(SPEC.md:465, 633).

Mesh I/O is pinned to the reference's OWN load_mesh/save_mesh, compiled
unmodified from /root/reference (oracle/ref_build): identical face tables,
switches and bytes written; identical config_error messages.  The matrix
writers are checked against the CPU oracle's export (values <= 1e-12
normwise, indices bit-exact) and the Table-1 goldens.
"""
import ctypes as C
import os

import numpy as np
import pytest

from paper_1204_1533_b200 import CONFIGS, LDG_K11, LDG_K12, LDG_K21, Case

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libref_setup.so")


def _ref():
    if not os.path.exists(REF_SO):
        if os.path.isdir("/root/reference/proj/src"):
            import subprocess

            subprocess.check_call([os.path.join(ROOT, "oracle", "ref_build", "build.sh")])
        else:
            pytest.skip("reference tree not present")
    L = C.CDLL(REF_SO)
    if not hasattr(L, "ref_case_load"):
        pytest.skip("oracle/_ref predates the mesh I/O wrappers")
    vp, ip, dp = C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_double)
    L.ref_case_load.argtypes = [C.c_int, C.c_char_p, C.c_int, ip, dp]
    L.ref_case_load.restype = vp
    L.ref_case_save.argtypes = [vp, C.c_char_p]
    L.ref_case_free.argtypes = [vp]
    L.ref_case_num_faces.argtypes = [vp]
    L.ref_case_faces.argtypes = [vp, ip]
    L.ref_case_switches.argtypes = [vp, C.POINTER(C.c_int8)]
    L.ref_last_error.restype = C.c_char_p
    return L


def _periodic(length):
    return [((4, 2), (length[0], 0.0)), ((1, 3), (0.0, length[1]))]


def _ref_load(ref, p, path, periodic=()):
    pt = np.ascontiguousarray(np.asarray([t for t, _ in periodic], dtype=np.int32).reshape(-1, 2))
    tr = np.zeros((len(periodic), 3))
    for i, (_, t) in enumerate(periodic):
        tr[i, :2] = t
    return ref.ref_case_load(p, os.fsencode(path), len(periodic), pt.ctypes.data_as(C.POINTER(C.c_int32)),
                             tr.ctypes.data_as(C.POINTER(C.c_double)))


MESHES = [  # n, p, periodic, jitter, permute, rotate, length
    (5, 3, False, 0.2, True, True, (1.0, 1.0)),
    (6, 4, True, 0.15, True, True, (10.0, 10.0)),
    (4, 2, True, 0.1, False, False, (2.0, 1.0)),
]


@pytest.mark.parametrize("spec", MESHES, ids=[f"n{m[0]}p{m[1]}per{int(m[2])}" for m in MESHES])
def test_mesh_file_round_trip_matches_reference(tmp_path, spec):
    ref = _ref()
    n, p, periodic, jit, perm, rot, length = spec
    src = Case.lattice(2, n, p, (*length, 1.0), jit, periodic, False, perm, rot, seeds=(21, 22, 23))
    # the lattice's pre-pairing mesh file: vertices, elements, every boundary tag line
    path = tmp_path / "in.mesh"
    v, el, tags = src.vertices(), src.elements(), src.tag_lines()
    with open(path, "w") as f:
        f.write(f"{len(v)} {len(el)} {len(tags)}\n")
        for x, y in v:
            f.write(f"{float(x)!r} {float(y)!r}\n")
        for q in el:
            f.write(" ".join(str(int(a)) for a in q) + "\n")
        for e, lf, t in tags:
            f.write(f"{e} {lf} {t}\n")
    pairs = _periodic(length) if periodic else ()
    ours = Case.load_mesh(str(path), p, periodic=pairs)
    h = _ref_load(ref, p, str(path), pairs)
    assert h, ref.ref_last_error()
    try:
        nf = ref.ref_case_num_faces(h)
        rf = np.zeros(nf * 6, dtype=np.int32)
        ref.ref_case_faces(h, rf.ctypes.data_as(C.POINTER(C.c_int32)))
        assert np.array_equal(rf.reshape(nf, 6), ours.faces())
        assert np.array_equal(ours.faces(), src.faces())  # file path == in-memory lattice path
        sw = np.zeros(ours.E * 2, dtype=np.int8)
        ref.ref_case_switches(h, sw.ctypes.data_as(C.POINTER(C.c_int8)))
        assert np.array_equal(sw.reshape(ours.E, 2), ours.switches())
        assert np.array_equal(ours.jac, src.jac) and np.array_equal(ours.nvec, src.nvec)
        # save_mesh: byte-identical to the reference's writer
        a, b = tmp_path / "ours.mesh", tmp_path / "ref.mesh"
        ours.save_mesh(str(a))
        assert ref.ref_case_save(h, os.fsencode(str(b))) == 0
        assert a.read_bytes() == b.read_bytes()
    finally:
        ref.ref_case_free(h)
    # a saved (post-pairing) file loads back to the same faces
    back = Case.load_mesh(str(a), p)
    if not periodic:
        assert np.array_equal(back.faces(), ours.faces())
    else:
        assert back.faces()[:, 5].max() <= 4 and (back.faces()[:, 2] >= 0).sum() < ours.nf


BAD = [
    ("", "header"),
    ("3 1 0\n0 0\n1 0\n", "vertex 2"),
    ("4 1 0\n0 0\n1 0\n1 1\n0 1\n0 1 2\n", "element 0"),
    ("4 1 0\n0 0\n1 0\n1 1\n0 1\n0 1 2 7\n", "out of range"),
    ("4 1 1\n0 0\n1 0\n1 1\n0 1\n0 1 2 3\n0 5 1\n", "tag line 0"),
    ("6 2 1\n0 0\n1 0\n2 0\n0 1\n1 1\n2 1\n0 1 4 3\n1 2 5 4\n0 1 1\n", "not a boundary face"),
]


@pytest.mark.parametrize("text,needle", BAD, ids=[b[1].replace(" ", "_") for b in BAD])
def test_mesh_file_errors_match_reference(tmp_path, text, needle):
    from paper_1204_1533_b200.linedg import ConfigError

    ref = _ref()
    path = tmp_path / "bad.mesh"
    path.write_text(text)
    with pytest.raises(ConfigError) as ei:
        Case.load_mesh(str(path), 2)
    assert needle in str(ei.value)
    assert not _ref_load(ref, 2, str(path))
    assert str(ei.value) == ref.ref_last_error().decode()


def test_missing_mesh_file(tmp_path):
    from paper_1204_1533_b200.linedg import ConfigError

    with pytest.raises(ConfigError, match="cannot open"):
        Case.load_mesh(str(tmp_path / "nope.mesh"), 2)


# ------------------------------------------------------------ matrix export
def test_oracle_triplets_match_csc_and_table1():
    """The checker itself: the triplet list equals the oracle's CSC export
    (SPEC.md:391-394), and the sparsity row reproduces Table 1 (2p+5 node
    columns per row on a periodic 2-D mesh)."""
    from oracle.pyoracle import Oracle

    cfg = CONFIGS[1]
    case, U = cfg.build(n=4)
    ora = Oracle(case, cfg.physics)
    ora.assemble(U)
    i, j, v = ora.triplets(LDG_K11)
    colptr, rowidx, vals = ora.export_csc(LDG_K11)
    cj = np.repeat(np.arange(len(colptr) - 1), np.diff(colptr))
    o = np.lexsort((cj, rowidx))
    assert np.array_equal(rowidx[o], i) and np.array_equal(cj[o], j) and np.array_equal(vals[o], v)
    p, avg, nnz = ora.sparsity_row(LDG_K11)
    assert p == 4 and avg == 2 * 4 + 5 and nnz == case.E * case.npe * 13 * 16


def _read_triplets(path):
    a = np.loadtxt(path, dtype=np.float64, ndmin=2)
    return a[:, 0].astype(np.int64), a[:, 1].astype(np.int64), a[:, 2]


GPU_CASES = [(0, 4), (1, 3), (2, 3), (3, 2), (4, 2)]


@pytest.mark.gpu
@pytest.mark.parametrize("ci,n", GPU_CASES, ids=[f"C{c + 1}-n{n}" for c, n in GPU_CASES])
def test_gpu_triplets_and_csv_match_oracle(tmp_path, ci, n):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle.pyoracle import Oracle
    from paper_1204_1533_b200.linedg import LineDG

    cfg = CONFIGS[ci]
    case, U = cfg.build(n=n)
    gpu = LineDG(case, cfg.physics)
    ora = Oracle(case, cfg.physics)
    gpu.assemble_jacobians(torch.from_numpy(U).cuda())
    ora.assemble(U)
    mats = [LDG_K11] + ([LDG_K12, LDG_K21] if cfg.physics.second_order() else [])
    csv = tmp_path / "sparsity.csv"
    for k, which in enumerate(mats):
        path = tmp_path / f"k{which}.txt"
        gpu.write_triplets(which, str(path))
        i, j, v = _read_triplets(path)
        i0, j0, v0 = ora.triplets(which)
        assert np.array_equal(i, i0) and np.array_equal(j, j0), "triplet indices differ"
        assert np.abs(v - v0).max() <= 1e-12 * max(np.abs(v0).max(), 1e-300)
        # %.17g round-trips: the file holds the device values exactly
        _, _, vb = gpu.export_blocks(which)
        mask = ora.structural_mask(which)
        assert np.array_equal(np.sort(v), np.sort(vb[:, mask].ravel()))
        gpu.write_sparsity_csv(which, str(csv), append=k > 0)
    lines = csv.read_text().splitlines()
    assert lines[0] == "p,avg_cols_per_block_row,nnz" and len(lines) == 1 + len(mats)
    for line, which in zip(lines[1:], mats):
        p, avg, nnz = line.split(",")
        p0, avg0, nnz0 = ora.sparsity_row(which)
        assert int(p) == p0 and int(nnz) == nnz0 and abs(float(avg) - avg0) <= 5e-7


@pytest.mark.gpu
def test_gpu_triplets_need_an_assembled_jacobian(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1204_1533_b200.linedg import LineDG, SolverError

    cfg = CONFIGS[1]
    case, U = cfg.build(n=2)
    gpu = LineDG(case, cfg.physics)
    with pytest.raises(SolverError):
        gpu.write_triplets(LDG_K11, str(tmp_path / "x.txt"))
    with pytest.raises(ValueError):
        gpu.write_sparsity_csv(LDG_K12, str(tmp_path / "x.csv"))


@pytest.mark.parametrize("spec", MESHES[:2], ids=["n5p3", "n6p4"])
def test_refine_uniform_matches_reference(tmp_path, spec):
    """refine_uniform (mesh.cpp:168-213; element count x4 per
    refinement, tags inherited): vertices bitwise, elements, faces, switches
    and mapping equal to the reference's own implementation; twice -> x16."""
    ref = _ref()
    if not hasattr(ref, "ref_case_refine"):
        pytest.skip("oracle/_ref predates the refinement wrapper")
    vp, ip, dp = C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_double)
    ref.ref_case_refine.argtypes = [vp]
    ref.ref_case_refine.restype = vp
    ref.ref_case_num_vertices.argtypes = [vp]
    ref.ref_case_vertices.argtypes = [vp, dp]
    ref.ref_case_elements.argtypes = [vp, ip]
    n, p, _, jit, perm, rot, length = spec
    src = Case.lattice(2, n, p, (*length, 1.0), jit, False, False, perm, rot, seeds=(31, 32, 33))
    path = tmp_path / "in.mesh"
    src.save_mesh(str(path))
    ours0 = Case.load_mesh(str(path), p)
    h0 = _ref_load(ref, p, str(path))
    assert h0, ref.ref_last_error()
    try:
        ours, h = ours0, h0
        for level in (1, 2):
            ours = ours.refine()
            h2 = ref.ref_case_refine(h)
            assert h2, ref.ref_last_error()
            if h is not h0:
                ref.ref_case_free(h)
            h = h2
            assert ours.E == src.E * 4 ** level
            nv = ref.ref_case_num_vertices(h)
            rv = np.zeros(2 * nv)
            ref.ref_case_vertices(h, rv.ctypes.data_as(dp))
            assert np.array_equal(rv.reshape(nv, 2), ours.vertices())
            re_ = np.zeros(4 * ours.E, dtype=np.int32)
            ref.ref_case_elements(h, re_.ctypes.data_as(ip))
            assert np.array_equal(re_.reshape(-1, 4), ours.elements())
            nf = ref.ref_case_num_faces(h)
            rf = np.zeros(nf * 6, dtype=np.int32)
            ref.ref_case_faces(h, rf.ctypes.data_as(ip))
            assert np.array_equal(rf.reshape(nf, 6), ours.faces())
            sw = np.zeros(ours.E * 2, dtype=np.int8)
            ref.ref_case_switches(h, sw.ctypes.data_as(C.POINTER(C.c_int8)))
            assert np.array_equal(sw.reshape(ours.E, 2), ours.switches())
        if h is not h0:
            ref.ref_case_free(h)
    finally:
        ref.ref_case_free(h0)
