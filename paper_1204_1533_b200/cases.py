"""Seeded synthetic cases for the BASELINE.json configurations.

Every mesh, state and vector comes from the setup library (csrc/host) and a
splitmix64 stream with a recorded seed, so the GPU path, the oracle and the
CPU baseline all see bit-identical inputs.  The reference's public meshes are
not available; these lattice meshes with jitter, random
renumbering and (where BASELINE.json asks) random local orientation stand in
for them.  Choices BASELINE.json leaves open are fixed here and recorded in
DESIGN.md ("Config choices"), following SURVEY.md Appendix C.
"""
from __future__ import annotations

import ctypes as C
import os
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _abi
from ._abi import LdgBc, LdgPhysics, LhLatticeParams, dptr, host_lib

GAMMA = 1.4


@dataclass
class Physics:
    """Mirror of GasModel / LdgParams / BoundaryTable (physics.hpp:10-35,
    SPEC.md:197-205).  bcs: list of (tag, values) Dirichlet conditions or
    (tag, values, kind) with kind an ldg_bc_kind (LDG_BC_NEUMANN: values =
    g_N; LDG_BC_CHARACTERISTIC: values = far-field state; LDG_BC_SLIP_WALL:
    values unused)."""

    kind: int = _abi.LDG_EULER
    riemann: int = _abi.LDG_ROE
    gamma: float = GAMMA
    mu: float = 0.0
    prandtl: float = 0.72
    c11: float = 0.0
    c22: float = 0.0
    c11_bd: float = 1.0
    bcs: List[Tuple[int, Sequence[float]]] = field(default_factory=list)

    def components(self, dim: int) -> int:
        return 1 if self.kind == _abi.LDG_POISSON else dim + 2

    def second_order(self) -> bool:
        return self.kind == _abi.LDG_POISSON or (self.kind == _abi.LDG_NAVIER_STOKES and self.mu != 0.0)

    def to_c(self):
        arr = (LdgBc * max(1, len(self.bcs)))()
        for i, bc in enumerate(self.bcs):
            tag, vals = bc[0], bc[1]
            arr[i].tag = tag
            arr[i].kind = bc[2] if len(bc) > 2 else _abi.LDG_BC_DIRICHLET
            for k, v in enumerate(vals):
                arr[i].value[k] = v
        ph = LdgPhysics(self.kind, self.riemann, self.gamma, self.mu, self.prandtl, self.c11,
                        self.c22, self.c11_bd, len(self.bcs), arr)
        ph._keep = arr  # keep the array alive with the struct
        return ph


class Case:
    """Basis + mesh + switches + mapping of one configuration (the reference's
    NodalBasis1D, QuadMesh, SwitchAssignment, ElementMapping), flattened."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        self._lib = host_lib()
        self.setup_ptr = self._lib.lh_case_setup(self._h)
        s = self.setup_ptr.contents
        self.dim, self.p, self.nq, self.E, self.nf = s.dim, s.p, s.n_quad, s.n_elems, s.n_faces
        self.np = self.p + 1
        self.npe = self.np ** self.dim
        self.NL = self.np ** (self.dim - 1)

    # ------------------------------------------------------------ builders
    @classmethod
    def lattice(cls, dim: int, n: int, p: int, length=(1.0, 1.0, 1.0), jitter=0.0,
                periodic=False, jitter_boundary=False, permute=False, rotate=False,
                seeds=(1, 2, 3), gll=True) -> "Case":
        prm = LhLatticeParams(dim, n, p, 1 if gll else 0, (C.c_double * 3)(*length), jitter,
                              int(periodic), int(jitter_boundary), int(permute), int(rotate),
                              seeds[0], seeds[1], seeds[2])
        h = C.c_void_p()
        st = host_lib().lh_case_lattice(C.byref(prm), C.byref(h))
        if st != 0:
            raise _setup_error(st)
        return cls(h.value)

    @classmethod
    def custom(cls, dim: int, p: int, verts, elems, btags=(), periodic=(), gll=True) -> "Case":
        """Custom mesh: vertices (nv x dim), elements (ne x 2^dim), boundary
        tag lines (elem, local_face, tag) as in the reference text format
        (mesh.cpp:115-146), periodic pairs ((tag_a, tag_b), translation)."""
        v = np.ascontiguousarray(verts, dtype=np.float64)
        el = np.ascontiguousarray(elems, dtype=np.int32)
        bt = np.ascontiguousarray(np.asarray(btags, dtype=np.int32).reshape(-1, 3))
        pt = np.ascontiguousarray(np.asarray([t for t, _ in periodic], dtype=np.int32).reshape(-1, 2))
        ptr = np.zeros((len(periodic), 3))
        for i, (_, tr) in enumerate(periodic):
            ptr[i, :len(tr)] = tr
        h = C.c_void_p()
        st = host_lib().lh_case_custom(dim, p, 1 if gll else 0, v.shape[0], dptr(v), el.shape[0],
                                       _abi.iptr(el), bt.shape[0], _abi.iptr(bt), len(periodic),
                                       _abi.iptr(pt), dptr(ptr), C.byref(h))
        if st != 0:
            raise _setup_error(st)
        return cls(h.value)

    @classmethod
    def load_mesh(cls, path: str, p: int, periodic=(), gll=True) -> "Case":
        """Case from a reference mesh text file (load_mesh, mesh.cpp:115-146),
        then optional periodic pairs ((tag_a, tag_b), translation)."""
        pt = np.ascontiguousarray(np.asarray([t for t, _ in periodic], dtype=np.int32).reshape(-1, 2))
        ptr = np.zeros((len(periodic), 3))
        for i, (_, tr) in enumerate(periodic):
            ptr[i, :len(tr)] = tr
        h = C.c_void_p()
        st = host_lib().lh_case_load_mesh(os.fsencode(path), p, 1 if gll else 0, len(periodic),
                                          _abi.iptr(pt), dptr(ptr), C.byref(h))
        if st != 0:
            raise _setup_error(st)
        return cls(h.value)

    def refine(self, periodic=()) -> "Case":
        """Uniformly refined case (refine_uniform, mesh.cpp:168-213: each quad
        split into four), same basis, then optional periodic pairs."""
        pt = np.ascontiguousarray(np.asarray([t for t, _ in periodic], dtype=np.int32).reshape(-1, 2))
        ptr = np.zeros((len(periodic), 3))
        for i, (_, tr) in enumerate(periodic):
            ptr[i, :len(tr)] = tr
        h = C.c_void_p()
        st = self._lib.lh_case_refine(self._h, len(periodic), _abi.iptr(pt), dptr(ptr), C.byref(h))
        if st != 0:
            raise _setup_error(st)
        return Case(h.value)

    def save_mesh(self, path: str):
        """Write the mesh in the reference text format (save_mesh, mesh.cpp:148-160)."""
        st = self._lib.lh_case_save_mesh(self._h, os.fsencode(path))
        if st != 0:
            raise _setup_error(st)

    # ------------------------------------------------------ curved geometry
    def remap(self, projector):
        """Recompute the mapping with a boundary projection (the reference
        CurveProjector, mapping.hpp:13-15; mapping.cpp:30-65):
        projector(x, y, tag) -> (x', y') for every boundary-face node."""
        def _fn(_user, x, tag, out):
            px, py = projector(x[0], x[1], tag)
            out[0] = px
            out[1] = py

        cb = _abi.CURVE_FN(_fn)
        st = self._lib.lh_case_remap(self._h, cb, None)
        if st != 0:
            raise _setup_error(st)

    def remap_circles(self, circles):
        """Built-in projector: circles = [(tag, cx, cy, r), ...]; boundary faces
        with that tag are projected radially onto the circle."""
        n = len(circles)
        tags = np.array([c[0] for c in circles], dtype=np.int32)
        cx, cy, r = (np.array([c[k] for c in circles], dtype=np.float64) for k in (1, 2, 3))
        st = self._lib.lh_case_remap_circles(self._h, n, _abi.iptr(tags), dptr(cx), dptr(cy), dptr(r))
        if st != 0:
            raise _setup_error(st)

    def __del__(self):
        try:
            if self._h:
                self._lib.lh_case_free(self._h)
                self._h = None
        except Exception:
            pass

    # -------------------------------------------------------------- views
    def _arr(self, ptr, n, dtype=np.float64):
        if not ptr:
            return None
        return np.ctypeslib.as_array(ptr, shape=(n,)).view(dtype).copy()

    @property
    def coords(self) -> np.ndarray:
        s = self.setup_ptr.contents
        return self._arr(s.node_coords, self.E * self.npe * self.dim).reshape(self.E, self.npe, self.dim)

    @property
    def jac(self) -> np.ndarray:
        s = self.setup_ptr.contents
        return self._arr(s.jac_at_nodes, self.E * self.npe).reshape(self.E, self.npe)

    @property
    def nvec(self) -> np.ndarray:
        s = self.setup_ptr.contents
        D = self.dim
        return self._arr(s.nvec_quad, self.E * D * self.NL * self.nq * D).reshape(
            self.E, D, self.NL, self.nq, D)

    @property
    def normal_end(self) -> np.ndarray:
        s = self.setup_ptr.contents
        D = self.dim
        return self._arr(s.normal_end, self.E * D * 2 * self.NL * D).reshape(self.E, D, 2, self.NL, D)

    def faces(self) -> np.ndarray:
        """(n_faces, 6): elem_l, face_l, elem_r, face_r, orient, tag."""
        s = self.setup_ptr.contents
        cols = [s.face_elem_l, s.face_face_l, s.face_elem_r, s.face_face_r, s.face_orient, s.face_tag]
        return np.stack([np.ctypeslib.as_array(c, shape=(self.nf,)).copy() for c in cols], axis=1)

    def elem_face(self) -> np.ndarray:
        s = self.setup_ptr.contents
        return np.ctypeslib.as_array(s.elem_face, shape=(self.E * 2 * self.dim,)).copy().reshape(
            self.E, 2 * self.dim)

    def switches(self) -> np.ndarray:
        s = self.setup_ptr.contents
        return np.ctypeslib.as_array(s.switch_plus, shape=(self.E * self.dim,)).copy().reshape(
            self.E, self.dim)

    def vertices(self) -> np.ndarray:
        nv = self._lib.lh_case_num_vertices(self._h)
        return np.ctypeslib.as_array(self._lib.lh_case_vertices(self._h),
                                     shape=(nv * self.dim,)).copy().reshape(nv, self.dim)

    def elements(self) -> np.ndarray:
        vpe = 2 ** self.dim
        return np.ctypeslib.as_array(self._lib.lh_case_elements(self._h),
                                     shape=(self.E * vpe,)).copy().reshape(self.E, vpe)

    def tag_lines(self) -> np.ndarray:
        """(n, 3) boundary tag lines (elem, local_face, tag) of a lattice case,
        recorded before periodic pairing (the reference mesh-file form)."""
        n = self._lib.lh_case_num_tag_lines(self._h)
        out = np.zeros(3 * n, dtype=np.int32)
        if n:
            self._lib.lh_case_tag_lines(self._h, _abi.iptr(out))
        return out.reshape(n, 3)

    def switch_violations(self) -> int:
        return self._lib.lh_case_switch_violations(self._h)

    def num_boundary_faces(self) -> int:
        return self._lib.lh_case_num_boundary_faces(self._h)

    # ------------------------------------------------------------- states
    def fill(self, kind: int, m: int, prm: Sequence[float], seed: int) -> np.ndarray:
        out = np.zeros(self.E * self.npe * m)
        p = np.asarray(list(prm) + [0.0], dtype=np.float64)
        st = self._lib.lh_fill_state(self._h, kind, m, dptr(p), seed, dptr(out))
        if st != 0:
            raise _setup_error(st)
        return out

    def normal_vector(self, m: int, seed: int) -> np.ndarray:
        return self.fill(5, m, [], seed)


def _setup_error(st: int) -> Exception:
    msg = host_lib().lh_last_error().decode()
    from .linedg import ConfigError

    if st == _abi.LDG_ERR_CONFIG:
        return ConfigError(msg)
    if st == _abi.LDG_ERR_INVALID_ARGUMENT:
        return ValueError(msg)
    return RuntimeError(msg)


# ---------------------------------------------------------------- configs
@dataclass
class Config:
    """One BASELINE.json configuration (index 0..4 = C1..C5)."""

    index: int
    name: str
    dim: int
    n: int
    p: int
    length: Tuple[float, float, float]
    jitter: float
    periodic: bool
    permute: bool
    rotate: bool
    physics: Physics
    state_kind: int
    state_prm: Tuple[float, ...]
    source: Optional[str] = None

    def seeds(self):
        base = self.index + 1
        return (1000 + base, 2000 + base, 3000 + base)

    @property
    def state_seed(self) -> int:
        return 4000 + self.index + 1

    @property
    def vector_seed(self) -> int:
        return 5000 + self.index + 1

    def build(self, n: Optional[int] = None, rotate: Optional[bool] = None,
              p: Optional[int] = None) -> Tuple[Case, np.ndarray]:
        """Mesh + state.  n / rotate / p override for scaled-down parity cases."""
        case = Case.lattice(self.dim, n or self.n, p or self.p, self.length, self.jitter, self.periodic,
                            False, self.permute, self.rotate if rotate is None else rotate,
                            self.seeds())
        m = self.physics.components(self.dim)
        U = case.fill(self.state_kind, m, self.state_prm, self.state_seed)
        return case, U

    def source_for(self, case: Case) -> Optional[np.ndarray]:
        if self.source != "poisson_sin":
            return None
        X = case.coords.reshape(-1, case.dim)
        return 2.0 * math.pi ** 2 * np.sin(math.pi * X[:, 0]) * np.sin(math.pi * X[:, 1])

    def dofs(self) -> int:
        m = self.physics.components(self.dim)
        return (self.n ** self.dim) * (self.p + 1) ** self.dim * m


def _configs() -> List[Config]:
    tgv_mu = 1.0 * 0.1 * (1.0 / (2.0 * math.pi)) / 1600.0
    vortex = (5.0, 1.5, 0.5, math.atan2(1.0, 2.0), 5.0, 5.0, 1.0, 0.5, 1.0 / GAMMA, GAMMA, 0.0, 1e-3)
    return [
        Config(0, "C1 2-D Poisson p=3 32^2", 2, 32, 3, (1.0, 1.0, 1.0), 0.2, False, True, True,
               Physics(_abi.LDG_POISSON, _abi.LDG_ROE, c11_bd=1.0,
                       bcs=[(t, [0.0]) for t in (1, 2, 3, 4)]),
               1, (1e-3,), source="poisson_sin"),
        Config(1, "C2 2-D Euler p=4 128^2 (vortex, Roe)", 2, 128, 4, (10.0, 10.0, 1.0), 0.15, True, True,
               False, Physics(_abi.LDG_EULER, _abi.LDG_ROE), 2, vortex),
        Config(2, "C3 2-D Navier-Stokes p=4 256^2 (Re=1000, LDG)", 2, 256, 4, (1.0, 1.0, 1.0), 0.15, True,
               True, False, Physics(_abi.LDG_NAVIER_STOKES, _abi.LDG_ROE, mu=3e-4, prandtl=0.72), 3,
               (1.0, 0.3, 0.0, 1.0 / GAMMA, GAMMA, 1e-2, 8.0, 0.0)),
        Config(3, "C4 3-D Euler p=3 64^3 (Taylor-Green, LLF)", 3, 64, 3, (1.0, 1.0, 1.0), 0.1, True, True,
               True, Physics(_abi.LDG_EULER, _abi.LDG_LLF), 4,
               (0.1, 1.0, 1.0 / GAMMA, GAMMA, 2.0 * math.pi, 1e-3)),
        Config(4, "C5 3-D Navier-Stokes p=4 48^3 (Taylor-Green, Re=1600)", 3, 48, 4, (1.0, 1.0, 1.0), 0.1,
               True, True, False,
               Physics(_abi.LDG_NAVIER_STOKES, _abi.LDG_ROE, mu=tgv_mu, prandtl=0.71), 4,
               (0.1, 1.0, 1.0 / GAMMA, GAMMA, 2.0 * math.pi, 0.0)),
    ]


CONFIGS = _configs()


def annulus_mesh(nr: int, nt: int, r0: float, r1: float, stretch: float = 1.0):
    """Straight-sided quadrilaterals of the ring r0 <= r <= r1 around the origin
    (the paper's cylinder geometry): nr elements radially
    (geometric spacing ratio `stretch`), nt around, closed by vertex reuse.
    Returns (verts, elems, btags) with tag 1 on the cylinder (local face 3)
    and tag 2 on the far field (local face 1); elements CCW (v0 at (r_i,
    theta_j), v1 at (r_i+1, theta_j))."""
    if stretch == 1.0:
        radii = np.linspace(r0, r1, nr + 1)
    else:
        w = stretch ** np.arange(nr)
        radii = r0 + (r1 - r0) * np.concatenate([[0.0], np.cumsum(w) / w.sum()])
    th = 2 * np.pi * np.arange(nt) / nt
    verts = np.array([[r * np.cos(t), r * np.sin(t)] for t in th for r in radii])
    vid = lambda i, j: (j % nt) * (nr + 1) + i  # noqa: E731
    elems, btags = [], []
    for j in range(nt):
        for i in range(nr):
            e = len(elems)
            elems.append([vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)])
            if i == 0:
                btags.append([e, 3, 1])
            if i == nr - 1:
                btags.append([e, 1, 2])
    return verts, np.array(elems, dtype=np.int32), np.array(btags, dtype=np.int32)
