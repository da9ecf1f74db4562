"""Python mirror of the reference's hot-path API,
backed by the sm_100a library through its C-ABI (include/linedg_b200.h).

    ctx = LineDG(case, physics)                  # discretization context
    R = ctx.residual_first_order(U)
    Q = ctx.gradient_residual(U)
    R = ctx.residual_second_order(U, Q)
    R = ctx.residual_primal(U)
    ctx.assemble_jacobians(U)                    # SPEC.md:409 (Analytic)
    y = ctx.split_matvec(alpha_dt, v)

Device arguments are torch.float64 CUDA tensors in the reference GridFunction
layout (field.hpp:8-9); numpy arrays take the host path (H2D, kernels, D2H).
Errors are raised with the reference's taxonomy (errors.hpp:10-28).  There
is no CPU fallback: without the built library or a GPU the constructor
raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

from . import _abi
from ._abi import LdgPatternInfo, dptr, gpu_lib, iptr, lptr


class LineDGError(RuntimeError):
    pass


class PhysicalStateError(LineDGError):
    """physical_state_error (errors.hpp:10-18): carries the offending state."""

    def __init__(self, msg, state=None, elem=-1, node=-1):
        super().__init__(msg)
        self.state = state
        self.elem = elem
        self.node = node


class ConfigError(LineDGError):
    """config_error (errors.hpp:21-23)."""


class SolverError(LineDGError):
    """solver_error (errors.hpp:26-28)."""


class CudaError(LineDGError):
    pass


def _raise(status: int, msg: str, state=None, elem=-1, node=-1):
    if status == _abi.LDG_ERR_PHYSICAL_STATE:
        raise PhysicalStateError(msg, state, elem, node)
    if status == _abi.LDG_ERR_CONFIG:
        raise ConfigError(msg)
    if status == _abi.LDG_ERR_SOLVER:
        raise SolverError(msg)
    if status == _abi.LDG_ERR_CUDA:
        raise CudaError(msg)
    raise ValueError(msg)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


class LineDG:
    """Discretization context bound to one CUDA stream (the current torch
    stream unless given)."""

    def __init__(self, case, physics, stream=None):
        import torch

        self._torch = torch
        self.lib = gpu_lib()
        self.case = case
        self.physics = physics
        self._ph = physics.to_c()
        if stream is None:
            stream = torch.cuda.current_stream()
        self.stream = stream
        h = C.c_void_p()
        st = self.lib.ldg_create(case.setup_ptr, C.byref(self._ph), C.c_void_p(stream.cuda_stream),
                                 C.byref(h))
        if st != 0:
            _raise(st, self.lib.ldg_last_error(None).decode())
        self._h = h
        self.m = self.lib.ldg_components(h)
        self.dim = case.dim
        self.n_dofs = int(self.lib.ldg_num_dofs(h))
        self.second_order = physics.second_order()

    def close(self):
        if getattr(self, "_h", None):
            self.lib.ldg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- plumbing
    def _check(self, st: int):
        if st == 0:
            return
        msg = self.lib.ldg_last_error(self._h).decode()
        state = None
        elem = C.c_int32(-1)
        node = C.c_int32(-1)
        if st == _abi.LDG_ERR_PHYSICAL_STATE:
            buf = np.zeros(8)
            self.lib.ldg_last_error_state(self._h, C.byref(elem), C.byref(node), dptr(buf))
            state = buf[: self.m].copy()
        _raise(st, msg, state, elem.value, node.value)

    def _dev(self, n: int, out=None):
        """Device result buffer: `out` (a contiguous float64 CUDA tensor of n
        entries, e.g. a preallocated buffer reused inside a CUDA graph) or new."""
        if out is None:
            return self._torch.empty(n, dtype=self._torch.float64, device="cuda")
        if not (_is_torch(out) and out.dtype == self._torch.float64 and out.is_cuda and out.is_contiguous()
                and out.numel() == n):
            raise ValueError(f"out must be a contiguous float64 CUDA tensor of {n} entries")
        return out

    @staticmethod
    def _ptr(t):
        return C.c_void_p(t.data_ptr()) if t is not None else None

    def _as_dev(self, x):
        t = x if _is_torch(x) else self._torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()
        if t.dtype != self._torch.float64 or not t.is_cuda or not t.is_contiguous():
            raise ValueError("expected a contiguous float64 CUDA tensor")
        return t

    @property
    def handle(self):
        return self._h

    def set_sync_errors(self, on: bool):
        self._check(self.lib.ldg_set_sync_errors(self._h, 1 if on else 0))

    def set_option(self, option: int, value: int):
        """ldg_set_option (LDG_OPT_SPMV_ROW_ORDER, LDG_OPT_ZERO_COPY)."""
        self._check(self.lib.ldg_set_option(self._h, int(option), int(value)))

    def synchronize(self):
        self._check(self.lib.ldg_synchronize(self._h))

    def kernel_launches(self) -> int:
        return int(self.lib.ldg_kernel_launches(self._h))

    def jacobian_bytes(self) -> int:
        return int(self.lib.ldg_jacobian_bytes(self._h))

    def set_boundary_function(self, tag: int, fn):
        """Space/time-dependent boundary data for the condition on `tag`
        (the reference's std::function data, physics.hpp:20-31):
        fn(x, t) -> m values at the boundary end node x; None restores the
        constant ldg_bc values."""
        if not hasattr(self, "_bc_cbs"):
            self._bc_cbs = {}
        if fn is None:
            self._bc_cbs.pop(tag, None)
            self._check(self.lib.ldg_set_boundary_function(self._h, tag, _abi.BC_FN(), None))
            return
        cb = _abi.make_bc_fn(fn, self.dim, self.m)
        self._bc_cbs[tag] = cb  # keep the ctypes callback alive
        self._check(self.lib.ldg_set_boundary_function(self._h, tag, cb, None))

    def set_source(self, S: Optional[np.ndarray]):
        a = None if S is None else np.ascontiguousarray(S, dtype=np.float64)
        self._check(self.lib.ldg_set_source(self._h, dptr(a)))

    # ------------------------------------------------------------ residuals
    @staticmethod
    def _host_out(out, n):
        """Result array of a host-path call: `out` (e.g. pinned memory, so the
        device-to-host copy runs at full PCIe speed) or a new array."""
        if out is None:
            return np.empty(n)
        if not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.flags.c_contiguous and out.size == n):
            raise ValueError(f"out must be a contiguous float64 array of {n} entries")
        return out

    def residual(self, U, t: float = 0.0, Q_out=None, out=None):
        """dU/dt = R(U, D(U)) (first-order physics: R(U)).  Device tensors in,
        device tensor out; numpy in -> numpy out (host path, into `out` if given)."""
        if not _is_torch(U):
            Uh = np.ascontiguousarray(U, dtype=np.float64)
            R = self._host_out(out, self.n_dofs)
            Qh = np.empty(self.n_dofs * self.dim) if (Q_out is not None and self.second_order) else None
            self._check(self.lib.ldg_residual_host(self._h, dptr(Uh), t, dptr(R), dptr(Qh)))
            if Qh is not None:
                Q_out[...] = Qh
            return R
        U = self._as_dev(U)
        R = self._dev(self.n_dofs, out)
        self._check(self.lib.ldg_residual(self._h, self._ptr(U), t, self._ptr(R), self._ptr(Q_out)))
        return R

    residual_first_order = residual
    residual_primal = residual

    def gradient_residual(self, U, t: float = 0.0):
        U = self._as_dev(U)
        Q = self._dev(self.n_dofs * self.dim)
        self._check(self.lib.ldg_gradient(self._h, self._ptr(U), t, self._ptr(Q)))
        return Q

    def residual_second_order(self, U, Q, t: float = 0.0):
        U = self._as_dev(U)
        Q = self._as_dev(Q)
        R = self._dev(self.n_dofs)
        self._check(self.lib.ldg_residual_uq(self._h, self._ptr(U), self._ptr(Q), t, self._ptr(R)))
        return R

    # ------------------------------------------------------------ Jacobians
    def assemble_jacobians(self, U, t: float = 0.0):
        if not _is_torch(U):
            Uh = np.ascontiguousarray(U, dtype=np.float64)
            self._check(self.lib.ldg_jacobian_assemble_host(self._h, dptr(Uh), t))
            return
        U = self._as_dev(U)
        self._check(self.lib.ldg_jacobian_assemble(self._h, self._ptr(U), t))

    def assemble_jacobians_q(self, U, Q, t: float = 0.0):
        """Assembly at U with the gradient Q = D(U) already on the device (from
        residual(U, Q_out=Q)): the Newton step's R and J share one gradient."""
        U = self._as_dev(U)
        Q = self._as_dev(Q) if self.second_order else None
        self._check(self.lib.ldg_jacobian_assemble_q(self._h, self._ptr(U), self._ptr(Q), t))

    def residual_and_assemble(self, U, t: float = 0.0, out=None, Q_out=None):
        """Host buffers: R(U) and the Jacobian at U from one upload of U
        (ldg_residual_assemble_host); returns R."""
        Uh = np.ascontiguousarray(U, dtype=np.float64)
        R = self._host_out(out, self.n_dofs)
        Qh = np.empty(self.n_dofs * self.dim) if (Q_out is not None and self.second_order) else None
        self._check(self.lib.ldg_residual_assemble_host(self._h, dptr(Uh), t, dptr(R), dptr(Qh)))
        if Qh is not None:
            Q_out[...] = Qh
        return R

    def pattern_info(self, which: int) -> LdgPatternInfo:
        info = LdgPatternInfo()
        self._check(self.lib.ldg_pattern_info_get(self._h, which, C.byref(info)))
        return info

    def export_blocks(self, which: int, elems: Optional[Sequence[int]] = None, values: bool = True):
        """(rows, cols, vals) of the node pattern in reference numbering,
        sorted by (row, col); vals: (nnzb, block_rows, block_cols)."""
        info = self.pattern_info(which)
        el = None if elems is None else np.ascontiguousarray(elems, dtype=np.int32)
        if el is None:
            nnzb = info.nnzb
        else:
            cnt = C.c_int64()
            self._check(self.lib.ldg_export_blocks_subset(self._h, which, iptr(el), len(el), None, None,
                                                          None, C.byref(cnt)))
            nnzb = cnt.value
        rows = np.empty(nnzb, dtype=np.int64)
        cols = np.empty(nnzb, dtype=np.int64)
        vals = np.empty(nnzb * info.block_rows * info.block_cols) if values else None
        cnt = C.c_int64()
        self._check(self.lib.ldg_export_blocks_subset(
            self._h, which, iptr(el), 0 if el is None else len(el), lptr(rows), lptr(cols), dptr(vals),
            C.byref(cnt)))
        if values:
            vals = vals.reshape(nnzb, info.block_rows, info.block_cols)
        return rows, cols, vals

    def write_triplets(self, which: int, path: str):
        """Text triplets `i j value` of one matrix."""
        self._check(self.lib.ldg_write_triplets(self._h, which, os.fsencode(path)))

    def write_sparsity_csv(self, which: int, path: str, append: bool = False):
        """Sparsity summary CSV `p,avg_cols_per_block_row,nnz`."""
        self._check(self.lib.ldg_write_sparsity_csv(self._h, which, os.fsencode(path), 1 if append else 0))

    def spmv(self, which: int, x, out=None):
        if not _is_torch(x):
            xh = np.ascontiguousarray(x, dtype=np.float64)
            ny = self.n_dofs * (self.dim if which == _abi.LDG_K21 else 1)
            y = self._host_out(out, ny)
            self._check(self.lib.ldg_bsr_spmv_host(self._h, which, dptr(xh), dptr(y)))
            return y
        x = self._as_dev(x)
        ny = self.n_dofs * (self.dim if which == _abi.LDG_K21 else 1)
        y = self._dev(ny, out)
        self._check(self.lib.ldg_bsr_spmv(self._h, which, self._ptr(x), self._ptr(y)))
        return y

    # ------------------------------------------------- preconditioned GMRES
    def set_precond_mode(self, mode: int):
        """Block-Jacobi mode: 0 LU solves (default), 1 explicit block inverses."""
        self._check(self.lib.ldg_set_precond_mode(self._h, mode))

    def precond_build(self, alpha_dt: float):
        """Block-Jacobi preconditioner of I - alpha_dt A~."""
        self._check(self.lib.ldg_precond_build(self._h, alpha_dt))

    def precond_apply(self, r, out=None):
        if not _is_torch(r):
            rh = np.ascontiguousarray(r, dtype=np.float64)
            z = self._host_out(out, self.n_dofs)
            self._check(self.lib.ldg_precond_apply_host(self._h, dptr(rh), dptr(z)))
            return z
        r = self._as_dev(r)
        z = self._dev(self.n_dofs)
        self._check(self.lib.ldg_precond_apply(self._h, self._ptr(r), self._ptr(z)))
        return z

    def gmres(self, alpha_dt: float, b, rtol: float = 1e-8, maxit: int = 50, restart: int = 30,
              precond: bool = True, out=None):
        """Right-preconditioned GMRES on (I - alpha_dt (K11 + K12 K21)) x = b:
        (x, iterations, converged, ||b - A x||)."""
        it = C.c_int32()
        cv = C.c_int32()
        rn = C.c_double()
        if not _is_torch(b):
            bh = np.ascontiguousarray(b, dtype=np.float64)
            x = self._host_out(out, self.n_dofs)
            self._check(self.lib.ldg_gmres_host(self._h, alpha_dt, dptr(bh), dptr(x), rtol, maxit, restart,
                                                1 if precond else 0, C.byref(it), C.byref(cv), C.byref(rn)))
            return x, it.value, bool(cv.value), rn.value
        b = self._as_dev(b)
        x = self._dev(self.n_dofs)
        self._check(self.lib.ldg_gmres(self._h, alpha_dt, self._ptr(b), self._ptr(x), rtol, maxit, restart,
                                       1 if precond else 0, C.byref(it), C.byref(cv), C.byref(rn)))
        return x, it.value, bool(cv.value), rn.value

    # ---------------------------------------------------- time integration
    def _state_on_device(self, U):
        """(device copy of U, came_from_host)."""
        if _is_torch(U):
            return self._as_dev(U).clone(), False
        import torch

        return torch.from_numpy(np.array(U, dtype=np.float64)).cuda(), True

    def rk4_step(self, U, dt: float, t: float = 0.0):
        """Classical RK4 step of dU/dt = R(U)."""
        Ud, host = self._state_on_device(U)
        self._check(self.lib.ldg_rk4_step(self._h, self._ptr(Ud), t, dt))
        return Ud.cpu().numpy() if host else Ud

    def dirk3_step(self, U, dt: float, cfg=None, t: float = 0.0):
        """L-stable DIRK3 step with Newton + (preconditioned) GMRES and Jacobian reuse
        (SPEC.md:501-523): (U_next, stats dict).  cfg: _abi.newton_cfg(...)."""
        cfg = cfg if cfg is not None else _abi.newton_cfg()
        Ud, host = self._state_on_device(U)
        st = _abi.LdgSolverStats()
        self._check(self.lib.ldg_dirk3_step(self._h, self._ptr(Ud), t, dt, C.byref(cfg), C.byref(st)))
        return (Ud.cpu().numpy() if host else Ud), st.as_dict()

    def steady_solve(self, U, cfg=None, t: float = 0.0):
        """Pseudo-transient continuation to R(U) = 0:
        (U_steady, stats dict).  cfg: _abi.steady_cfg(...)."""
        cfg = cfg if cfg is not None else _abi.steady_cfg()
        Ud, host = self._state_on_device(U)
        st = _abi.LdgSolverStats()
        self._check(self.lib.ldg_steady_solve(self._h, self._ptr(Ud), t, C.byref(cfg), C.byref(st)))
        return (Ud.cpu().numpy() if host else Ud), st.as_dict()

    def split_matvec(self, alpha_dt: float, v, out=None):
        """(I - alpha_dt (K11 + K12 K21)) v without forming the product."""
        if not _is_torch(v):
            vh = np.ascontiguousarray(v, dtype=np.float64)
            y = self._host_out(out, self.n_dofs)
            self._check(self.lib.ldg_split_matvec_host(self._h, alpha_dt, dptr(vh), dptr(y)))
            return y
        v = self._as_dev(v)
        y = self._dev(self.n_dofs, out)
        self._check(self.lib.ldg_split_matvec(self._h, alpha_dt, self._ptr(v), self._ptr(y)))
        return y
