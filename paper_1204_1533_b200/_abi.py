"""ctypes declarations of the C-ABI in include/linedg_b200.h and of the setup
library (csrc/host/lh_capi.cpp).  The shared libraries are built in-tree
(``make`` / ``__graft_entry__.build()``) and loaded from this directory."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))

LDG_OK = 0
LDG_ERR_PHYSICAL_STATE = 1
LDG_ERR_CONFIG = 2
LDG_ERR_SOLVER = 3
LDG_ERR_CUDA = 4
LDG_ERR_INVALID_ARGUMENT = 5

LDG_POISSON, LDG_EULER, LDG_NAVIER_STOKES = 0, 1, 2
LDG_ROE, LDG_LLF = 0, 1
LDG_BC_DIRICHLET = 0
LDG_BC_NEUMANN = 1
LDG_BC_CHARACTERISTIC = 2
LDG_BC_SLIP_WALL = 3
LDG_BC_NO_SLIP_ADIABATIC = 4
LDG_K11, LDG_K12, LDG_K21 = 0, 1, 2
LDG_OPT_SPMV_ROW_ORDER, LDG_OPT_ZERO_COPY = 1, 2

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)


class LdgBc(C.Structure):
    _fields_ = [("tag", C.c_int32), ("kind", C.c_int32), ("value", C.c_double * 8)]


class LdgPhysics(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("riemann", C.c_int32),
        ("gamma", C.c_double),
        ("mu", C.c_double),
        ("prandtl", C.c_double),
        ("c11", C.c_double),
        ("c22", C.c_double),
        ("c11_bd", C.c_double),
        ("n_bc", C.c_int32),
        ("bcs", C.POINTER(LdgBc)),
    ]


class LdgSetup(C.Structure):
    _fields_ = [
        ("dim", C.c_int32),
        ("p", C.c_int32),
        ("n_quad", C.c_int32),
        ("n_elems", C.c_int32),
        ("n_faces", C.c_int32),
        ("nodes", _dp),
        ("quad_points", _dp),
        ("quad_weights", _dp),
        ("phi_at_quad", _dp),
        ("dphi_at_quad", _dp),
        ("mass", _dp),
        ("face_elem_l", _ip),
        ("face_face_l", _ip),
        ("face_elem_r", _ip),
        ("face_face_r", _ip),
        ("face_orient", _ip),
        ("face_tag", _ip),
        ("elem_face", _ip),
        ("switch_plus", C.POINTER(C.c_int8)),
        ("jac_at_nodes", _dp),
        ("nvec_quad", _dp),
        ("normal_end", _dp),
        ("node_coords", _dp),
    ]


class LdgPatternInfo(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("nnzb", C.c_int64), ("block_rows", C.c_int32),
                ("block_cols", C.c_int32)]


class LhLatticeParams(C.Structure):
    _fields_ = [
        ("dim", C.c_int32),
        ("n", C.c_int32),
        ("p", C.c_int32),
        ("gll", C.c_int32),
        ("length", C.c_double * 3),
        ("jitter", C.c_double),
        ("periodic", C.c_int32),
        ("jitter_boundary", C.c_int32),
        ("permute", C.c_int32),
        ("rotate", C.c_int32),
        ("seed_jitter", C.c_uint64),
        ("seed_perm", C.c_uint64),
        ("seed_rot", C.c_uint64),
    ]


# CurveProjector callback: fn(user, x[2], tag, out[2]) (mapping.hpp:13-15)
CURVE_FN = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_double))


# Boundary-data callback: fn(user, x[dim], t, out[m]) (ldg_bc_fn; physics.hpp:20-31)
BC_FN = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(C.c_double), C.c_double, C.POINTER(C.c_double))


def make_bc_fn(fn, dim: int, m: int):
    """ctypes callback from fn(x: tuple of dim floats, t) -> sequence of m values."""
    def _cb(_user, x, t, out):
        v = fn(tuple(x[d] for d in range(dim)), t)
        for k in range(m):
            out[k] = float(v[k])
    return BC_FN(_cb)


def _load(name: str) -> C.CDLL:
    path = os.path.join(_HERE, name)
    if name == "liblinedg_b200.so" and os.environ.get("LDG_B200_LIB"):
        path = os.environ["LDG_B200_LIB"]  # A/B experiments with a variant build
    if not os.path.exists(path):
        raise RuntimeError(
            f"{name} is not built ({path}); run `make -j` or __graft_entry__.build() first")
    return C.CDLL(path)


_host = None
_gpu = None


def host_lib() -> C.CDLL:
    """The setup library (basis, mesh, mapping, generators)."""
    global _host
    if _host is None:
        L = _load("liblinedg_host.so")
        L.lh_last_error.restype = C.c_char_p
        L.lh_case_lattice.argtypes = [C.POINTER(LhLatticeParams), C.POINTER(C.c_void_p)]
        L.lh_case_custom.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, _dp, C.c_int32, _ip,
                                     C.c_int32, _ip, C.c_int32, _ip, _dp, C.POINTER(C.c_void_p)]
        L.lh_case_free.argtypes = [C.c_void_p]
        L.lh_case_load_mesh.argtypes = [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, _ip, _dp,
                                        C.POINTER(C.c_void_p)]
        L.lh_case_save_mesh.argtypes = [C.c_void_p, C.c_char_p]
        L.lh_case_refine.argtypes = [C.c_void_p, C.c_int32, _ip, _dp, C.POINTER(C.c_void_p)]
        L.lh_case_remap.argtypes = [C.c_void_p, CURVE_FN, C.c_void_p]
        L.lh_case_remap_circles.argtypes = [C.c_void_p, C.c_int32, _ip, _dp, _dp, _dp]
        L.lh_case_setup.argtypes = [C.c_void_p]
        L.lh_case_setup.restype = C.POINTER(LdgSetup)
        L.lh_case_num_vertices.argtypes = [C.c_void_p]
        L.lh_case_vertices.argtypes = [C.c_void_p]
        L.lh_case_vertices.restype = _dp
        L.lh_case_elements.argtypes = [C.c_void_p]
        L.lh_case_elements.restype = _ip
        L.lh_case_switch_violations.argtypes = [C.c_void_p]
        L.lh_case_num_boundary_faces.argtypes = [C.c_void_p]
        L.lh_case_num_tag_lines.argtypes = [C.c_void_p]
        L.lh_case_tag_lines.argtypes = [C.c_void_p, _ip]
        L.lh_case_tag_lines.restype = None
        L.lh_basis.argtypes = [C.c_int32, C.c_int32] + [_dp] * 8
        L.lh_gauss_legendre.argtypes = [C.c_int32, _dp, _dp]
        L.lh_fill_state.argtypes = [C.c_void_p, C.c_int32, C.c_int32, _dp, C.c_uint64, _dp]
        _host = L
    return _host


class LdgNewtonCfg(C.Structure):
    """ldg_newton_cfg (include/linedg_b200.h)."""
    _fields_ = [("gmres_iters", C.c_int32), ("recompute_threshold", C.c_int32), ("max_newton", C.c_int32),
                ("use_precond", C.c_int32), ("newton_tol", C.c_double)]


class LdgSolverStats(C.Structure):
    """ldg_solver_stats (include/linedg_b200.h)."""
    _fields_ = [("newton_iters", C.c_int32), ("gmres_iters", C.c_int32), ("jacobian_assemblies", C.c_int32),
                ("residual_evals", C.c_int32), ("residual_norm", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class LdgSteadyCfg(C.Structure):
    """ldg_steady_cfg (include/linedg_b200.h)."""
    _fields_ = [("dt0", C.c_double), ("growth", C.c_double), ("n_steps", C.c_int32), ("dt_final", C.c_double),
                ("gmres_iters", C.c_int32), ("gmres_rtol", C.c_double), ("recompute_threshold", C.c_int32),
                ("max_newton", C.c_int32), ("use_precond", C.c_int32), ("newton_tol", C.c_double),
                ("log_csv", C.c_char_p)]


def steady_cfg(dt0=1e-2, growth=2.0, n_steps=10, dt_final=0.0, gmres_iters=30, gmres_rtol=1e-3,
               recompute_threshold=1, max_newton=20, use_precond=True, newton_tol=1e-10, log_csv=None):
    """Pseudo-transient continuation policy (geometric ramp
    dt0 * 2^k over 10 steps, then Newton without the time derivative)."""
    return LdgSteadyCfg(dt0, growth, n_steps, dt_final, gmres_iters, gmres_rtol, recompute_threshold, max_newton,
                        1 if use_precond else 0, newton_tol, None if log_csv is None else os.fsencode(log_csv))


def newton_cfg(gmres_iters=5, recompute_threshold=15, max_newton=50, use_precond=True, newton_tol=1e-8):
    """The paper's Newton/GMRES policy."""
    return LdgNewtonCfg(gmres_iters, recompute_threshold, max_newton, 1 if use_precond else 0, newton_tol)


GPU_SYMBOLS = [
    "ldg_create", "ldg_destroy", "ldg_last_error", "ldg_last_error_state", "ldg_components",
    "ldg_num_dofs", "ldg_set_source", "ldg_residual", "ldg_residual_uq", "ldg_gradient",
    "ldg_jacobian_assemble", "ldg_pattern_info_get", "ldg_bsr_spmv", "ldg_split_matvec",
    "ldg_export_blocks", "ldg_export_blocks_subset", "ldg_set_sync_errors", "ldg_synchronize",
    "ldg_residual_host", "ldg_jacobian_assemble_host", "ldg_bsr_spmv_host", "ldg_split_matvec_host",
    "ldg_kernel_launches", "ldg_jacobian_bytes",
    "ldg_precond_build", "ldg_precond_apply", "ldg_precond_apply_host", "ldg_gmres", "ldg_gmres_host",
    "ldg_rk4_step", "ldg_dirk3_step", "ldg_write_triplets", "ldg_write_sparsity_csv", "ldg_steady_solve",
    "ldg_set_boundary_function", "ldg_set_precond_mode", "ldg_set_option", "ldg_jacobian_assemble_q",
    "ldg_residual_assemble_host", "ldg_gradient_host", "ldg_residual_uq_host",
]


def gpu_lib() -> C.CDLL:
    """The sm_100a hot-path library.  There is no CPU fallback: loading fails
    loudly when the library is missing, and ldg_create fails without a GPU."""
    global _gpu
    if _gpu is None:
        L = _load("liblinedg_b200.so")
        vp = C.c_void_p
        L.ldg_create.argtypes = [C.POINTER(LdgSetup), C.POINTER(LdgPhysics), vp, C.POINTER(vp)]
        L.ldg_destroy.argtypes = [vp]
        L.ldg_destroy.restype = None
        L.ldg_last_error.argtypes = [vp]
        L.ldg_last_error.restype = C.c_char_p
        L.ldg_last_error_state.argtypes = [vp, _ip, _ip, _dp]
        L.ldg_components.argtypes = [vp]
        L.ldg_num_dofs.argtypes = [vp]
        L.ldg_num_dofs.restype = C.c_int64
        L.ldg_set_source.argtypes = [vp, _dp]
        L.ldg_residual.argtypes = [vp, vp, C.c_double, vp, vp]
        L.ldg_residual_uq.argtypes = [vp, vp, vp, C.c_double, vp]
        L.ldg_gradient.argtypes = [vp, vp, C.c_double, vp]
        L.ldg_jacobian_assemble.argtypes = [vp, vp, C.c_double]
        L.ldg_jacobian_assemble_q.argtypes = [vp, vp, vp, C.c_double]
        L.ldg_pattern_info_get.argtypes = [vp, C.c_int, C.POINTER(LdgPatternInfo)]
        L.ldg_bsr_spmv.argtypes = [vp, C.c_int, vp, vp]
        L.ldg_split_matvec.argtypes = [vp, C.c_double, vp, vp]
        L.ldg_export_blocks.argtypes = [vp, C.c_int, _lp, _lp, _dp]
        L.ldg_export_blocks_subset.argtypes = [vp, C.c_int, _ip, C.c_int32, _lp, _lp, _dp, _lp]
        L.ldg_set_sync_errors.argtypes = [vp, C.c_int]
        L.ldg_synchronize.argtypes = [vp]
        L.ldg_residual_host.argtypes = [vp, _dp, C.c_double, _dp, _dp]
        L.ldg_jacobian_assemble_host.argtypes = [vp, _dp, C.c_double]
        L.ldg_residual_assemble_host.argtypes = [vp, _dp, C.c_double, _dp, _dp]
        L.ldg_bsr_spmv_host.argtypes = [vp, C.c_int, _dp, _dp]
        L.ldg_split_matvec_host.argtypes = [vp, C.c_double, _dp, _dp]
        L.ldg_precond_build.argtypes = [vp, C.c_double]
        L.ldg_precond_apply.argtypes = [vp, vp, vp]
        L.ldg_precond_apply_host.argtypes = [vp, _dp, _dp]
        _g = [vp, C.c_double, vp, vp, C.c_double, C.c_int32, C.c_int32, C.c_int32,
              C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_double)]
        L.ldg_gmres.argtypes = _g
        L.ldg_gmres_host.argtypes = [vp, C.c_double, _dp, _dp] + _g[4:]
        L.ldg_rk4_step.argtypes = [vp, vp, C.c_double, C.c_double]
        L.ldg_dirk3_step.argtypes = [vp, vp, C.c_double, C.c_double, C.POINTER(LdgNewtonCfg),
                                     C.POINTER(LdgSolverStats)]
        L.ldg_set_precond_mode.argtypes = [vp, C.c_int]
        L.ldg_set_option.argtypes = [vp, C.c_int, C.c_int64]
        L.ldg_set_boundary_function.argtypes = [vp, C.c_int32, BC_FN, vp]
        L.ldg_steady_solve.argtypes = [vp, vp, C.c_double, C.POINTER(LdgSteadyCfg), C.POINTER(LdgSolverStats)]
        L.ldg_write_triplets.argtypes = [vp, C.c_int, C.c_char_p]
        L.ldg_write_sparsity_csv.argtypes = [vp, C.c_int, C.c_char_p, C.c_int]
        L.ldg_kernel_launches.argtypes = [vp]
        L.ldg_kernel_launches.restype = C.c_int64
        L.ldg_jacobian_bytes.argtypes = [vp]
        L.ldg_jacobian_bytes.restype = C.c_int64
        _gpu = L
    return _gpu


def dptr(a) -> "C._Pointer":
    """ctypes double* of a contiguous float64 numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


def iptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(_ip)


def lptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(_lp)
