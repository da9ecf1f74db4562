"""TEST INFRASTRUCTURE ONLY -- Python handle on the CPU oracle
(oracle/liblinedg_oracle.so, built from oracle/oracle.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this module.  It is the parity checker, never the thing measured or
shipped.  The oracle restates the reference's hot-path operations whose
sources are absent from the reference tree (see oracle/oracle.cpp header);
it is pinned by the SPEC.md known-answer tests and the Table-1 integer
goldens (tests/test_oracle_kats.py) and, for the setup inputs, by the
reference's own basis/mesh/mapping sources compiled against an Eigen shim
(oracle/ref_build, tests/test_setup_vs_reference.py).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "liblinedg_oracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"oracle library not built: {path} (run make)")
        L = C.CDLL(path)
        vp = C.c_void_p
        L.lo_last_error.restype = C.c_char_p
        L.lo_last_error_state.argtypes = [_dp, C.POINTER(C.c_int32)]
        L.lo_set_threads.argtypes = [C.c_int32]
        L.lo_set_threads.restype = None
        L.lo_max_threads.restype = C.c_int32
        L.lo_create.argtypes = [vp, vp, C.POINTER(vp)]
        L.lo_destroy.argtypes = [vp]
        L.lo_destroy.restype = None
        L.lo_components.argtypes = [vp]
        L.lo_set_source.argtypes = [vp, _dp]
        L.lo_gradient.argtypes = [vp, _dp, C.c_double, _dp]
        L.lo_residual_uq.argtypes = [vp, _dp, _dp, C.c_double, _dp]
        L.lo_residual.argtypes = [vp, _dp, C.c_double, _dp, _dp, _ip, C.c_int32]
        L.lo_residual_ext.argtypes = [vp, _dp, C.c_double, _dp, _ip, C.c_int32]
        L.lo_time_sample.argtypes = [vp, _dp, _dp, C.c_double, C.c_int32, _ip, C.c_int32, C.c_int32,
                                     C.c_int32, _dp]
        L.lo_assemble.argtypes = [vp, _dp, C.c_double, _ip, C.c_int32]
        L.lo_assemble_uq.argtypes = [vp, _dp, _dp]
        L.lo_pattern_info.argtypes = [vp, C.c_int32, _lp, _ip, _ip]
        L.lo_export_blocks.argtypes = [vp, C.c_int32, _lp, _lp, _dp]
        L.lo_export_csc.argtypes = [vp, C.c_int32, _lp, _lp, _dp, _lp]
        L.lo_spmv.argtypes = [vp, C.c_int32, _dp, _dp]
        L.lo_split_matvec.argtypes = [vp, C.c_double, _dp, _dp]
        L.lo_fd_dense.argtypes = [vp, C.c_int32, _dp, _dp, _dp]
        from paper_1204_1533_b200._abi import LdgNewtonCfg, LdgSolverStats, LdgSteadyCfg
        L.lo_rk4_step.argtypes = [vp, _dp, C.c_double, C.c_double]
        L.lo_dirk3_step.argtypes = [vp, _dp, C.c_double, C.c_double, C.POINTER(LdgNewtonCfg),
                                    C.POINTER(LdgSolverStats)]
        L.lo_steady_solve.argtypes = [vp, _dp, C.c_double, C.POINTER(LdgSteadyCfg), C.POINTER(LdgSolverStats)]
        L.lo_flop_model.argtypes = [vp, _dp]
        from paper_1204_1533_b200._abi import BC_FN
        L.lo_set_boundary_function.argtypes = [vp, C.c_int32, BC_FN, vp]
        L.lo_precond_build.argtypes = [vp, C.c_double]
        L.lo_set_precond_mode.argtypes = [vp, C.c_int32]
        L.lo_precond_apply.argtypes = [vp, _dp, _dp]
        L.lo_gmres.argtypes = [vp, C.c_double, _dp, C.c_double, C.c_int32, C.c_int32, C.c_int32, _dp,
                               C.POINTER(C.c_int32), C.POINTER(C.c_int32), _dp]
        L.lo_euler_flux.argtypes = [C.c_int32, _dp, C.c_double, _dp]
        L.lo_riemann.argtypes = [C.c_int32, C.c_int32, _dp, _dp, _dp, C.c_double, _dp]
        L.lo_ns_viscous_flux.argtypes = [C.c_int32, _dp, _dp, C.c_double, C.c_double, C.c_double, _dp]
        _lib = L
    return _lib


class OraclePhysicalStateError(RuntimeError):
    def __init__(self, msg, state):
        super().__init__(msg)
        self.state = state


def _d(a):
    return None if a is None else a.ctypes.data_as(_dp)


class Oracle:
    def __init__(self, case, physics):
        self.L = lib()
        self.case = case
        self._ph = physics.to_c()
        h = C.c_void_p()
        self._check(self.L.lo_create(C.cast(case.setup_ptr, C.c_void_p), C.cast(C.pointer(self._ph), C.c_void_p),
                                     C.byref(h)))
        self.h = h
        self.m = self.L.lo_components(h)
        self.dim = case.dim
        self.n_dofs = case.E * case.npe * self.m

    def __del__(self):
        try:
            if self.h:
                self.L.lo_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def _check(self, st):
        if st == 0:
            return
        msg = self.L.lo_last_error().decode()
        if st == 1:
            buf = np.zeros(8)
            n = C.c_int32()
            self.L.lo_last_error_state(_d(buf), C.byref(n))
            raise OraclePhysicalStateError(msg, buf[: n.value].copy())
        raise RuntimeError(f"oracle status {st}: {msg}")

    @staticmethod
    def set_threads(n: int):
        lib().lo_set_threads(n)

    @staticmethod
    def max_threads() -> int:
        return lib().lo_max_threads()

    def set_source(self, S):
        a = None if S is None else np.ascontiguousarray(S, dtype=np.float64)
        self._check(self.L.lo_set_source(self.h, _d(a)))

    def residual(self, U, t=0.0, elems: Optional[Sequence[int]] = None, want_q=False):
        U = np.ascontiguousarray(U, dtype=np.float64)
        R = np.zeros(self.n_dofs)
        Q = np.zeros(self.n_dofs * self.dim) if want_q else None
        el = None if elems is None else np.ascontiguousarray(elems, dtype=np.int32)
        self._check(self.L.lo_residual(self.h, _d(U), t, _d(R), _d(Q),
                                       None if el is None else el.ctypes.data_as(_ip),
                                       0 if el is None else len(el)))
        return (R, Q) if want_q else R

    def residual_ext(self, U, t=0.0, elems: Optional[Sequence[int]] = None):
        """The residual evaluated in x87 long double (64-bit significand) and
        rounded once: the accuracy yardstick for ill-conditioned states."""
        U = np.ascontiguousarray(U, dtype=np.float64)
        R = np.zeros(self.n_dofs)
        el = None if elems is None else np.ascontiguousarray(elems, dtype=np.int32)
        self._check(self.L.lo_residual_ext(self.h, _d(U), t, _d(R),
                                           None if el is None else el.ctypes.data_as(_ip),
                                           0 if el is None else len(el)))
        return R

    def time_sample(self, U, v, adt, nmv, elems, threads, reps=3):
        """CPU baseline sample: median seconds of (gradient, residual, Jacobian,
        nmv matvecs) over the elements `elems` (lo_time_sample)."""
        U = np.ascontiguousarray(U, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        el = np.ascontiguousarray(elems, dtype=np.int32)
        secs = np.zeros(4)
        self._check(self.L.lo_time_sample(self.h, _d(U), _d(v), adt, nmv, el.ctypes.data_as(_ip), len(el),
                                          threads, reps, _d(secs)))
        return secs

    def gradient(self, U, t=0.0):
        U = np.ascontiguousarray(U, dtype=np.float64)
        Q = np.zeros(self.n_dofs * self.dim)
        self._check(self.L.lo_gradient(self.h, _d(U), t, _d(Q)))
        return Q

    def residual_uq(self, U, Q, t=0.0):
        U = np.ascontiguousarray(U, dtype=np.float64)
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        R = np.zeros(self.n_dofs)
        self._check(self.L.lo_residual_uq(self.h, _d(U), _d(Q), t, _d(R)))
        return R

    def assemble(self, U, t=0.0, elems: Optional[Sequence[int]] = None):
        U = np.ascontiguousarray(U, dtype=np.float64)
        el = None if elems is None else np.ascontiguousarray(elems, dtype=np.int32)
        self._check(self.L.lo_assemble(self.h, _d(U), t, None if el is None else el.ctypes.data_as(_ip),
                                       0 if el is None else len(el)))

    def assemble_uq(self, U, Q):
        U = np.ascontiguousarray(U, dtype=np.float64)
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        self._check(self.L.lo_assemble_uq(self.h, _d(U), _d(Q)))

    def export_blocks(self, which):
        nnzb = C.c_int64()
        br = C.c_int32()
        bc = C.c_int32()
        self._check(self.L.lo_pattern_info(self.h, which, C.byref(nnzb), C.byref(br), C.byref(bc)))
        rows = np.empty(nnzb.value, dtype=np.int64)
        cols = np.empty(nnzb.value, dtype=np.int64)
        vals = np.empty(nnzb.value * br.value * bc.value)
        self._check(self.L.lo_export_blocks(self.h, which, rows.ctypes.data_as(_lp), cols.ctypes.data_as(_lp),
                                            _d(vals)))
        return rows, cols, vals.reshape(nnzb.value, br.value, bc.value)

    def structural_mask(self, which):
        """Structural scalar entries of a node block (the wire-format rule of
        ldg_write_triplets): K11 all; K12 all but the Navier-Stokes density
        row; K21 the component diagonal."""
        br = self.m * self.dim if which == 2 else self.m
        bc = self.m * self.dim if which == 1 else self.m
        mask = np.ones((br, bc), dtype=bool)
        if which == 1 and self._ph.kind == 2:
            mask[0, :] = False
        if which == 2:
            mask[:] = False
            for c in range(self.m):
                mask[c * self.dim:(c + 1) * self.dim, c] = True
        return mask

    def triplets(self, which):
        """(i, j, v) scalar triplets in the order ldg_write_triplets emits them
        (rows ascending; within a row, columns ascending) -- checker for the
        `i j value` export."""
        rows, cols, vals = self.export_blocks(which)
        mask = self.structural_mask(which)
        br, bc = mask.shape
        a, b = np.nonzero(mask)
        i = (rows[:, None] * br + a[None, :]).ravel()
        j = (cols[:, None] * bc + b[None, :]).ravel()
        v = vals[:, a, b].ravel()
        o = np.lexsort((j, i))
        return i[o], j[o], v[o]

    def sparsity_row(self, which):
        """(p, avg node-cols per node row, structural scalar nnz)."""
        rows, _, _ = self.export_blocks(which)
        n_rows = self.case.E * self.case.npe
        return self.case.p, len(rows) / n_rows, len(rows) * int(self.structural_mask(which).sum())

    def export_csc(self, which):
        nnz = C.c_int64()
        self._check(self.L.lo_export_csc(self.h, which, None, None, None, C.byref(nnz)))
        nnzb = C.c_int64()
        br = C.c_int32()
        bc = C.c_int32()
        self._check(self.L.lo_pattern_info(self.h, which, C.byref(nnzb), C.byref(br), C.byref(bc)))
        ncols = self.case.E * self.case.npe * bc.value
        colptr = np.zeros(ncols + 1, dtype=np.int64)
        rowidx = np.zeros(nnz.value, dtype=np.int64)
        vals = np.zeros(nnz.value)
        self._check(self.L.lo_export_csc(self.h, which, colptr.ctypes.data_as(_lp), rowidx.ctypes.data_as(_lp),
                                         _d(vals), None))
        return colptr, rowidx, vals

    def spmv(self, which, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        ny = self.n_dofs * (self.dim if which == 2 else 1)
        y = np.zeros(ny)
        self._check(self.L.lo_spmv(self.h, which, _d(x), _d(y)))
        return y

    def split_matvec(self, adt, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        y = np.zeros(self.n_dofs)
        self._check(self.L.lo_split_matvec(self.h, adt, _d(v), _d(y)))
        return y

    def set_precond_mode(self, mode):
        self._check(self.L.lo_set_precond_mode(self.h, mode))

    def precond_build(self, adt):
        self._check(self.L.lo_precond_build(self.h, adt))

    def precond_apply(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.zeros(self.n_dofs)
        self._check(self.L.lo_precond_apply(self.h, _d(r), _d(z)))
        return z

    def gmres(self, adt, b, rtol=1e-8, maxit=50, restart=30, precond=True):
        """(x, iterations, converged, ||b - A x||) of right-preconditioned GMRES."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(self.n_dofs)
        it = C.c_int32()
        cv = C.c_int32()
        rn = C.c_double()
        self._check(self.L.lo_gmres(self.h, adt, _d(b), rtol, maxit, restart, 1 if precond else 0, _d(x),
                                    C.byref(it), C.byref(cv), C.byref(rn)))
        return x, it.value, bool(cv.value), rn.value

    def rk4_step(self, U, dt, t=0.0):
        U = np.array(U, dtype=np.float64)
        self._check(self.L.lo_rk4_step(self.h, _d(U), t, dt))
        return U

    def dirk3_step(self, U, dt, cfg, t=0.0):
        """(U_next, stats dict); cfg = paper_1204_1533_b200._abi.newton_cfg(...)."""
        from paper_1204_1533_b200._abi import LdgSolverStats
        U = np.array(U, dtype=np.float64)
        st = LdgSolverStats()
        self._check(self.L.lo_dirk3_step(self.h, _d(U), t, dt, C.byref(cfg), C.byref(st)))
        return U, st.as_dict()

    def steady_solve(self, U, cfg, t=0.0):
        """(U_steady, stats dict); cfg = paper_1204_1533_b200._abi.steady_cfg(...)."""
        from paper_1204_1533_b200._abi import LdgSolverStats
        U = np.array(U, dtype=np.float64)
        st = LdgSolverStats()
        self._check(self.L.lo_steady_solve(self.h, _d(U), t, C.byref(cfg), C.byref(st)))
        return U, st.as_dict()

    def set_boundary_function(self, tag, fn):
        """fn(x, t) -> m values; None restores the constant data."""
        from paper_1204_1533_b200._abi import BC_FN, make_bc_fn
        if not hasattr(self, "_bc_cbs"):
            self._bc_cbs = {}
        if fn is None:
            self._bc_cbs.pop(tag, None)
            self._check(self.L.lo_set_boundary_function(self.h, tag, BC_FN(), None))
            return
        cb = make_bc_fn(fn, self.dim, self.m)
        self._bc_cbs[tag] = cb
        self._check(self.L.lo_set_boundary_function(self.h, tag, cb, None))

    def flop_model(self):
        """Algorithmic FP64 flops per element: {'residual', 'jacobian', 'spmv'}
        plus the per-evaluation flux counts (oracle lo_flop_model)."""
        out = np.zeros(7)
        self._check(self.L.lo_flop_model(self.h, _d(out)))
        keys = ("residual", "jacobian", "spmv", "flux", "riemann", "viscous_flux", "riemann_jacobian")
        return dict(zip(keys, out.tolist()))

    def fd_dense(self, which, U, Q=None):
        U = np.ascontiguousarray(U, dtype=np.float64)
        Qa = None if Q is None else np.ascontiguousarray(Q, dtype=np.float64)
        nu = self.n_dofs
        nrows = nu * self.dim if which == 2 else nu
        ncols = nu * self.dim if which == 1 else nu
        out = np.zeros(nrows * ncols)
        self._check(self.L.lo_fd_dense(self.h, which, _d(U), _d(Qa), _d(out)))
        return out.reshape(nrows, ncols)

    def dense(self, which):
        """Dense scalar matrix from the assembled blocks."""
        rows, cols, vals = self.export_blocks(which)
        br, bc = vals.shape[1], vals.shape[2]
        nr = self.case.E * self.case.npe * br
        nc = self.case.E * self.case.npe * bc
        A = np.zeros((nr, nc))
        for r, c, v in zip(rows, cols, vals):
            A[r * br:(r + 1) * br, c * bc:(c + 1) * bc] += v
        return A
