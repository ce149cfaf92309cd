"""Python mirror of the reference's solver-facing API, backed by libsdgpu.so.

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/core/include/sdc/*.hpp) so parity tests read like the
reference's own tests:

=========================  ================================================
this module                reference (proj/core/...)
=========================  ================================================
SparseMatrix               include/sdc/sparse.hpp:17-46
spmv / spmv_add            src/sparse.cpp:81-108
LinearOperator.from_matrix include/sdc/operator.hpp:18-28
Preconditioner             include/sdc/operator.hpp:34-62
IdentityPreconditioner     include/sdc/operator.hpp:64-76
sor_sweep                  src/precond.cpp:92-108
gauss_seidel_apply         src/precond.cpp:110-116
AmgOptions / AmgPreconditioner  include/sdc/precond.hpp:64-120
UzawaConfig / UzawaPreconditioner  include/sdc/precond.hpp:122-155
BlockPreconditioner        include/sdc/precond.hpp:162-199
ground_dof                 src/precond.cpp:375-392
RestartController          include/sdc/krylov.hpp:23-47
pd_gmres / bicgstab        src/krylov.cpp:47-292
power_iteration            src/krylov.cpp:307-339
assemble_monolithic        src/assembly.cpp:327-380 (n x n free-flow box)
=========================  ================================================

Errors: SDG_EDIM -> ValueError (std::invalid_argument), SDG_ESINGULAR /
SDG_EBREAKDOWN -> RuntimeError (std::runtime_error), CUDA failures ->
SdgCudaError.  There is no CPU fallback: if the CUDA library is missing or no
GPU is visible, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import threading
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsdgpu.so")

SDG_OK, SDG_EDIM, SDG_ESINGULAR, SDG_EBREAKDOWN, SDG_ECUDA, SDG_ENOMEM, SDG_ENCCL, SDG_EINVAL = range(8)


class SdgCudaError(RuntimeError):
    """CUDA runtime / library failure inside libsdgpu.so."""


_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_vp = C.c_void_p
_i = C.c_int
_d = C.c_double
_i64 = C.c_int64


class _Restart(C.Structure):
    _fields_ = [("m_init", _i), ("m_min", _i), ("m_step", _i), ("m_max", _i), ("current_m", _i),
                ("previous_rate", _d), ("has_rate_sample", _i), ("alpha_p", _d), ("alpha_d", _d),
                ("stall_threshold", _d)]


class _Report(C.Structure):
    _fields_ = [("iterations", _i), ("converged", _i), ("wall_time", _d), ("final_residual", _d),
                ("residual_history", C.POINTER(_d)), ("history_capacity", _i), ("history_length", _i),
                ("precond_applications", _i64), ("device_ms", _d), ("breakdown", _i)]


class _AmgOpts(C.Structure):
    _fields_ = [("max_levels", _i), ("strength_theta", _d), ("coarse_threshold", _i),
                ("components", C.POINTER(_i))]


class _UzawaOpts(C.Structure):
    _fields_ = [("amg", _AmgOpts), ("power_tol_rel", _d), ("power_max_iters", _i), ("power_seed", C.c_uint),
                ("omega_override", _d)]


class _Scenario(C.Structure):
    _fields_ = [("n", _i), ("permeability", _d), ("alpha_bj", _d), ("nu", _d), ("rho", _d), ("dt", _d),
                ("t_end", _d), ("dp_max", _d), ("t", _d)]


_lib = None
_lib_lock = threading.Lock()


def lib():
    """Load libsdgpu.so (fails loudly: there is no CPU fallback)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2108_13229_b200.build`")
        L = C.CDLL(LIB_PATH)

        def p(name, res, args):
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args

        P = C.POINTER
        p("sdg_last_error", C.c_char_p, [])
        p("sdg_version", C.c_char_p, [])
        p("sdg_restart_defaults", None, [P(_Restart)])
        p("sdg_amg_defaults", None, [P(_AmgOpts)])
        p("sdg_uzawa_defaults", None, [P(_UzawaOpts)])
        p("sdg_context_create", _i, [_i, P(_vp)])
        p("sdg_context_destroy", _i, [_vp])
        p("sdg_context_synchronize", _i, [_vp])
        p("sdg_context_stream", _vp, [_vp])
        p("sdg_context_launches", _i64, [_vp])
        p("sdg_context_set_profiling", _i, [_vp, _i])
        p("sdg_context_profile", _i, [_vp, _i, P(_i64), P(_d), P(_d)])
        p("sdg_profile_family_name", C.c_char_p, [_i])
        p("sdg_matrix_create", _i, [_vp, _i, _i, _ip, _ip, _dp, P(_vp)])
        p("sdg_matrix_destroy", _i, [_vp])
        p("sdg_matrix_rows", _i, [_vp])
        p("sdg_matrix_cols", _i, [_vp])
        p("sdg_matrix_nnz", _i64, [_vp])
        p("sdg_spmv", _i, [_vp, _dp, _dp])
        p("sdg_spmv_add", _i, [_vp, _dp, _dp, _d])
        p("sdg_spmv_device", _i, [_vp, _vp, _vp])
        p("sdg_sor_sweep", _i, [_vp, _dp, _dp, _d])
        p("sdg_amg_create", _i, [_vp, P(_AmgOpts), P(_vp)])
        p("sdg_uzawa_create", _i, [_vp, _vp, _vp, P(_UzawaOpts), P(_vp)])
        p("sdg_block_create", _i, [_i, _vp, _i, _i, _i, _vp, _vp, P(_vp)])
        p("sdg_identity_create", _i, [_vp, _i, P(_vp)])
        p("sdg_ilu0_create", _i, [_vp, P(_vp)])
        p("sdg_ground_dof_host", _i, [_i, _ip, _ip, _dp, _i])
        p("sdg_gs_merged_sweep_host", _i, [_i, _ip, _ip, _dp, _i, _i, _dp, _vp, _dp, P(_i)])
        p("sdg_galerkin_device", _i, [_vp, _i, _ip, _ip, _dp, _ip, _i, _vp, _vp, _vp, P(_i64)])
        p("sdg_lu_factor", _i, [_vp, _i, _ip, _ip, _dp, P(_vp)])
        p("sdg_lu_solve", _i, [_vp, _dp, _dp])
        p("sdg_lu_info", _i, [_vp, P(_i), P(_i), P(_i64)])
        p("sdg_lu_destroy", None, [_vp])
        p("sdg_nd_solve_host", _i, [_i, _ip, _ip, _dp, _i, _i, _vp, _vp, _vp, P(_i), P(_i), P(_i), P(_i64), _vp, _i])
        p("sdg_td_create", _i, [_vp, _i, _i, _i, _i, _i, _i, _i, _d, P(_vp)])
        p("sdg_precond_destroy", _i, [_vp])
        p("sdg_precond_rows", _i, [_vp])
        p("sdg_precond_apply", _i, [_vp, _dp, _dp])
        p("sdg_precond_apply_device", _i, [_vp, _vp, _vp])
        p("sdg_precond_applications", _i64, [_vp])
        p("sdg_precond_setup_memory_doubles", _i64, [_vp])
        p("sdg_precond_work_per_apply", _i64, [_vp])
        p("sdg_precond_omega", _d, [_vp])
        p("sdg_precond_setup_seconds", _d, [_vp])
        p("sdg_precond_hierarchy", _i, [_vp, _i, P(_i), P(_i), P(_i64), _i])
        p("sdg_precond_features", _i, [_vp, P(_i)])
        p("sdg_precond_set_graphs", _i, [_vp, _i])
        p("sdg_pd_gmres", _i, [_vp, _vp, _dp, _dp, _d, _i, P(_Restart), P(_Report)])
        p("sdg_pd_gmres_device", _i, [_vp, _vp, _vp, _vp, _d, _i, P(_Restart), P(_Report)])
        p("sdg_pd_gmres_warm", _i, [_vp, _vp, _dp, _dp, _d, _i, P(_Restart), P(_Report)])
        p("sdg_pd_gmres_warm_device", _i, [_vp, _vp, _vp, _vp, _d, _i, P(_Restart), P(_Report)])
        p("sdg_bicgstab", _i, [_vp, _vp, _dp, _dp, _d, _i, P(_Report)])
        p("sdg_bicgstab_warm", _i, [_vp, _vp, _dp, _dp, _d, _i, P(_Report)])
        p("sdg_bicgstab_warm_device", _i, [_vp, _vp, _vp, _vp, _d, _i, P(_Report)])
        p("sdg_bicgstab_device", _i, [_vp, _vp, _vp, _vp, _d, _i, P(_Report)])
        p("sdg_power_iteration", _i, [_vp, _d, _i, C.c_uint, P(_d), P(_i), P(_i)])
        p("sdg_assemble_rhs_device", _i, [_vp, P(_Scenario), _vp, _vp])
        p("sdg_assemble_matrix_device", _i, [_vp, P(_Scenario), _vp, _vp, _vp, _vp, _i64, P(_i64)])
        p("sdg_assemble_monolithic", _i, [P(_Scenario), _vp, _vp, P(_i), P(_i64), P(_i), P(_i), P(_i),
                                          P(_i), _vp, _vp, _vp, _vp])
        p("sdg_assemble_stokes", _i, [P(_Scenario), _vp, _vp, P(_i), P(_i64), _vp, _vp, _vp, _vp])
        p("sdg_assemble_darcy", _i, [P(_Scenario), _vp, P(_i), P(_i64), _vp, _vp, _vp, _vp])
        p("sdg_stokes_pressure_trace", _i, [P(_Scenario), _dp, _dp])
        p("sdg_darcy_velocity_trace", _i, [P(_Scenario), _dp, _dp, _dp])
        p("sdg_host_hierarchy_build", _i, [_i, _ip, _ip, _dp, P(_AmgOpts), P(_vp)])
        p("sdg_host_hierarchy_levels", _i, [_vp])
        p("sdg_host_hierarchy_level", _i, [_vp, _i, P(_i), P(_i64), P(_i), P(_i), _vp, _vp, _vp, _vp])
        p("sdg_host_hierarchy_destroy", None, [_vp])
        _lib = L
        return L


def _check(rc: int):
    if rc == SDG_OK:
        return
    msg = lib().sdg_last_error().decode()
    if rc == SDG_EDIM:
        raise ValueError(msg)
    if rc in (SDG_ESINGULAR, SDG_EBREAKDOWN):
        raise RuntimeError(msg)
    if rc in (SDG_ECUDA, SDG_ENOMEM, SDG_ENCCL):
        raise SdgCudaError(msg)
    raise ValueError(msg)


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64)


def _i32(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.int32)


# ---------------------------------------------------------------------------
# context


class Context:
    """One CUDA device + stream; every handle created from it uses its stream."""

    def __init__(self, device: int = 0):
        self.h = _vp()
        _check(lib().sdg_context_create(device, C.byref(self.h)))
        self.device = device

    def synchronize(self):
        _check(lib().sdg_context_synchronize(self.h))

    @property
    def stream(self) -> int:
        return lib().sdg_context_stream(self.h) or 0

    @property
    def launches(self) -> int:
        return lib().sdg_context_launches(self.h)

    def set_profiling(self, enable: bool):
        _check(lib().sdg_context_set_profiling(self.h, int(enable)))

    def profile(self) -> dict:
        """Per kernel family: launches, total CUDA-event ms, total algorithmic bytes."""
        out = {}
        for f in range(15):  # PF_COUNT (common.hpp)
            n, ms, by = _i64(), _d(), _d()
            _check(lib().sdg_context_profile(self.h, f, C.byref(n), C.byref(ms), C.byref(by)))
            if n.value:
                out[lib().sdg_profile_family_name(f).decode()] = {"launches": n.value, "ms": ms.value,
                                                                   "bytes": by.value}
        return out

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib is not None:
            _lib.sdg_context_destroy(h)
            self.h = None


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ---------------------------------------------------------------------------
# sparse matrices


class SparseMatrix:
    """CSR matrix with the reference's field names (sparse.hpp:17-46).

    Host arrays; the device copy is created on first use and cached.
    """

    def __init__(self, n_rows: int = 0, n_cols: int = 0, row_offsets=None, col_indices=None, values=None):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.row_offsets = _i32(row_offsets if row_offsets is not None else np.zeros(self.n_rows + 1))
        self.col_indices = _i32(col_indices if col_indices is not None else [])
        self.values = _f64(values if values is not None else [])
        self._dev = None

    def nnz(self) -> int:
        return int(self.values.size)

    def row_cols(self, i):
        return self.col_indices[self.row_offsets[i]:self.row_offsets[i + 1]]

    def row_vals(self, i):
        return self.values[self.row_offsets[i]:self.row_offsets[i + 1]]

    def at(self, i, j) -> float:
        cols = self.row_cols(i)
        k = np.searchsorted(cols, j)
        if k < cols.size and cols[k] == j:
            return float(self.row_vals(i)[k])
        return 0.0

    @staticmethod
    def identity(n: int) -> "SparseMatrix":
        return SparseMatrix(n, n, np.arange(n + 1), np.arange(n), np.ones(n))

    @staticmethod
    def from_dense(d) -> "SparseMatrix":
        d = np.asarray(d, dtype=np.float64)
        rp, ci, vv = [0], [], []
        for i in range(d.shape[0]):
            nz = np.nonzero(d[i])[0]
            ci.extend(nz.tolist())
            vv.extend(d[i, nz].tolist())
            rp.append(len(ci))
        return SparseMatrix(d.shape[0], d.shape[1], rp, ci, vv)

    @staticmethod
    def from_coo(n_rows, n_cols, entries: Sequence[tuple]) -> "SparseMatrix":
        """CooBuilder semantics (sparse.cpp:55-79): stable sort, sum duplicates in insertion order."""
        order = sorted(range(len(entries)), key=lambda k: (entries[k][0], entries[k][1]))
        rp = [0] * (n_rows + 1)
        ci, vv = [], []
        k = 0
        for i in range(n_rows):
            while k < len(order) and entries[order[k]][0] == i:
                col = entries[order[k]][1]
                s = 0.0
                while k < len(order) and entries[order[k]][0] == i and entries[order[k]][1] == col:
                    s += entries[order[k]][2]
                    k += 1
                ci.append(col)
                vv.append(s)
            rp[i + 1] = len(ci)
        return SparseMatrix(n_rows, n_cols, rp, ci, vv)

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.n_rows, self.n_cols))
        for i in range(self.n_rows):
            s, e = self.row_offsets[i], self.row_offsets[i + 1]
            d[i, self.col_indices[s:e]] += self.values[s:e]
        return d

    def device(self, ctx: Optional[Context] = None) -> "DeviceMatrix":
        ctx = ctx or default_context()
        if self._dev is None or self._dev.ctx is not ctx:
            self._dev = DeviceMatrix(ctx, self)
        return self._dev


class DeviceMatrix:
    """sdg_matrix handle: the device copy of a SparseMatrix."""

    def __init__(self, ctx: Context, a: SparseMatrix):
        self.ctx = ctx
        self.n_rows, self.n_cols = a.n_rows, a.n_cols
        self.h = _vp()
        _check(lib().sdg_matrix_create(ctx.h, a.n_rows, a.n_cols, a.row_offsets, a.col_indices,
                                       a.values if a.values.size else np.zeros(1), C.byref(self.h)))

    def nnz(self) -> int:
        return lib().sdg_matrix_nnz(self.h)

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib is not None:
            _lib.sdg_matrix_destroy(h)
            self.h = None


def spmv(a: SparseMatrix, x) -> np.ndarray:
    """y = A x (sparse.cpp:81-90)."""
    x = _f64(x)
    if x.size != a.n_cols:
        raise ValueError("spmv: dimension mismatch")
    y = np.empty(a.n_rows)
    _check(lib().sdg_spmv(a.device().h, x if x.size else np.zeros(1), y if y.size else np.zeros(1)))
    return y


def spmv_add(a: SparseMatrix, x, y, alpha: float = 1.0) -> np.ndarray:
    """Returns y + alpha A x (sparse.cpp:98-108)."""
    x, y = _f64(x), _f64(y).copy()
    if x.size != a.n_cols or y.size != a.n_rows:
        raise ValueError("spmv_add: dimension mismatch")
    _check(lib().sdg_spmv_add(a.device().h, x, y, alpha))
    return y


def submatrix(a: SparseMatrix, row_begin, row_end, col_begin, col_end) -> SparseMatrix:
    """sparse.cpp:110-127 (host helper): rows [row_begin, row_end), columns
    [col_begin, col_end), entries kept in their row order."""
    if row_begin < 0 or row_end > a.n_rows or col_begin < 0 or col_end > a.n_cols or row_begin > row_end \
            or col_begin > col_end:
        raise ValueError("submatrix: bad range")
    nr = row_end - row_begin
    lo, hi = int(a.row_offsets[row_begin]), int(a.row_offsets[row_end])
    cols = a.col_indices[lo:hi]
    vals = a.values[lo:hi]
    counts = np.diff(a.row_offsets[row_begin:row_end + 1])
    row_id = np.repeat(np.arange(nr), counts)
    m = (cols >= col_begin) & (cols < col_end)
    rp = np.zeros(nr + 1, np.int64)
    rp[1:] = np.cumsum(np.bincount(row_id[m], minlength=nr))
    return SparseMatrix(nr, col_end - col_begin, rp, cols[m] - col_begin, vals[m])


def ground_dof(a: SparseMatrix, dof: int = 0) -> SparseMatrix:
    """precond.cpp:375-392."""
    vals = a.values.copy()
    _check(lib().sdg_ground_dof_host(a.n_rows, a.row_offsets, a.col_indices, vals, dof))
    return SparseMatrix(a.n_rows, a.n_cols, a.row_offsets.copy(), a.col_indices.copy(), vals)


def gs_merged_sweep_host(a: SparseMatrix, r, k: int, dyn_cap: int = 0, z_old=None):
    """Host check of the smoother's level merging (gs.cu merge_levels): one
    forward Gauss-Seidel sweep (omega = 1) in the merged form the device walk
    evaluates, groups of k dependency levels (dyn_cap > 0: dynamic groups).
    Returns (z_new, number of groups).  Runs without a GPU."""
    r = _f64(r)
    if r.size != a.n_rows or a.n_rows != a.n_cols:
        raise ValueError("gs_merged_sweep_host: dimension mismatch")
    zo = None if z_old is None else _f64(z_old).copy()
    z = np.zeros(a.n_rows)
    g = C.c_int(0)
    _check(lib().sdg_gs_merged_sweep_host(a.n_rows, a.row_offsets, a.col_indices, a.values, int(k), int(dyn_cap), r,
                                          None if zo is None else zo.ctypes.data, z, C.byref(g)))
    return z, g.value


def galerkin_product_device(a: SparseMatrix, aggregate_of, n_coarse: int, ctx: Optional[Context] = None) -> SparseMatrix:
    """galerkin_product (precond.cpp:177-185) on the GPU: A_c = P^T A P of an
    aggregation, bitwise the reference's sum order (csrc/galerkin.cu)."""
    ctx = ctx or default_context()
    agg = _i32(aggregate_of)
    if agg.size != a.n_rows:
        raise ValueError("galerkin_product: aggregate map length mismatch")
    rp = np.empty(n_coarse + 1, np.int32)
    ci = np.empty(max(a.nnz(), 1), np.int32)
    vv = np.empty(max(a.nnz(), 1), np.float64)
    nnz = _i64()
    _check(lib().sdg_galerkin_device(ctx.h, a.n_rows, a.row_offsets, a.col_indices,
                                     a.values if a.values.size else np.zeros(1), agg, int(n_coarse),
                                     rp.ctypes.data, ci.ctypes.data, vv.ctypes.data, C.byref(nnz)))
    return SparseMatrix(n_coarse, n_coarse, rp, ci[:nnz.value].copy(), vv[:nnz.value].copy())


class LUFactorization:
    """lu_factor / lu_solve (lu.hpp:38-41) on the GPU: the direct solve the AMG
    hierarchies use on their coarsest level (csrc/coarse.hpp)."""

    def __init__(self, a: SparseMatrix, ctx: Optional[Context] = None):
        if a.n_rows != a.n_cols:
            raise ValueError("lu_factor: matrix must be square")
        self.ctx = ctx or default_context()
        self.n = a.n_rows
        self.h = _vp()
        _check(lib().sdg_lu_factor(self.ctx.h, a.n_rows, a.row_offsets, a.col_indices,
                                   a.values if a.values.size else np.zeros(1), C.byref(self.h)))

    def rows(self) -> int:
        return self.n

    def solve(self, b) -> np.ndarray:
        b = _f64(b)
        if b.size != self.n:
            raise ValueError("lu_solve: dimension mismatch")
        x = np.empty(self.n)
        if self.n:
            _check(lib().sdg_lu_solve(self.h, b, x))
        return x

    def info(self) -> dict:
        d, k, s = _i(), _i(), _i64()
        _check(lib().sdg_lu_info(self.h, C.byref(d), C.byref(k), C.byref(s)))
        return {"dense": bool(d.value), "depth": k.value, "stored_doubles": s.value}

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().sdg_lu_destroy(self.h)
                self.h = None
        except Exception:
            pass


def lu_factor(a: SparseMatrix, ctx: Optional[Context] = None) -> LUFactorization:
    return LUFactorization(a, ctx)


def lu_solve(f: LUFactorization, b) -> np.ndarray:
    return f.solve(b)


def nd_solve_host(a: SparseMatrix, b=None, leaf_rows: int = 1024, max_depth: int = 32):
    """Host check of the coarse direct solve (csrc/coarse.hpp, replaces
    lu_factor/lu_solve lu.cpp:91-203): nested-dissection order of `a` and, when
    b is given, A^{-1} b through the block elimination.  Returns a dict with
    x, perm (new -> old), nodes (lo, mid, hi, depth per node, post-order),
    depth, max_separator and stored_doubles."""
    n = a.n_rows
    perm = np.empty(max(n, 1), np.int32)
    nn, dep, ms, sd = _i(), _i(), _i(), _i64()
    x = None
    if b is not None:
        b = _f64(b)
        if b.size != n:
            raise ValueError("nd_solve_host: dimension mismatch")
        x = np.empty(n)
    cap = 4 * max(1, n)
    nodes = np.empty((cap, 4), np.int32)
    _check(lib().sdg_nd_solve_host(n, a.row_offsets, a.col_indices, a.values, int(leaf_rows), int(max_depth),
                                   None if b is None else b.ctypes.data, None if x is None else x.ctypes.data,
                                   perm.ctypes.data, C.byref(nn), C.byref(dep), C.byref(ms), C.byref(sd),
                                   nodes.ctypes.data, cap))
    return {"x": x, "perm": perm[:n], "nodes": nodes[:nn.value].copy(), "depth": dep.value,
            "max_separator": ms.value, "stored_doubles": sd.value}


def sor_sweep(a: SparseMatrix, z, r, omega: float) -> np.ndarray:
    """One forward SOR sweep (precond.cpp:92-108); returns the updated z."""
    z, r = _f64(z).copy(), _f64(r)
    if z.size != a.n_rows or r.size != a.n_rows or a.n_rows != a.n_cols:
        raise ValueError("sor_sweep: dimension mismatch")
    if a.n_rows == 0:
        return z
    _check(lib().sdg_sor_sweep(a.device().h, z, r, omega))
    return z


def gauss_seidel_apply(a: SparseMatrix, r, omega: float = 1.0, sweeps: int = 1) -> np.ndarray:
    z = np.zeros(a.n_rows)
    for _ in range(sweeps):
        z = sor_sweep(a, z, r, omega)
    return z


# ---------------------------------------------------------------------------
# operator / preconditioners


class LinearOperator:
    """operator.hpp:18-28; device-backed when built from a matrix."""

    def __init__(self, n: int, apply_fn=None, matrix: Optional[SparseMatrix] = None):
        self.n = n
        self._fn = apply_fn
        self.matrix = matrix

    @staticmethod
    def from_matrix(a: SparseMatrix) -> "LinearOperator":
        return LinearOperator(a.n_rows, None, a)

    def apply(self, x) -> np.ndarray:
        if self.matrix is not None:
            return spmv(self.matrix, x)
        return np.asarray(self._fn(_f64(x)), dtype=np.float64)


class Preconditioner:
    """operator.hpp:34-62 over an sdg_precond handle."""

    def __init__(self, h, ctx: Context, keep=()):
        self.h = h
        self.ctx = ctx
        self._keep = list(keep)  # sub-handles / arrays that must outlive this one

    def rows(self) -> int:
        return lib().sdg_precond_rows(self.h)

    def apply(self, r) -> np.ndarray:
        r = _f64(r)
        if r.size != self.rows():
            raise ValueError("preconditioner: dimension mismatch")
        z = np.empty_like(r)
        _check(lib().sdg_precond_apply(self.h, r, z))
        return z

    def applications(self) -> int:
        return lib().sdg_precond_applications(self.h)

    def setup_memory_doubles(self) -> int:
        return lib().sdg_precond_setup_memory_doubles(self.h)

    def work_per_apply(self) -> int:
        return lib().sdg_precond_work_per_apply(self.h)

    def setup_seconds(self) -> float:
        return lib().sdg_precond_setup_seconds(self.h)

    def features(self) -> set:
        """Fast paths this handle runs: {"split", "early", "wave_v", "wave_d", "lattice_v", "lattice_d"}."""
        f = _i()
        _check(lib().sdg_precond_features(self.h, C.byref(f)))
        names = {1: "split", 2: "early", 4: "wave_v", 8: "wave_d", 16: "lattice_v", 32: "lattice_d"}
        return {nm for bit, nm in names.items() if f.value & bit}

    def hierarchy(self, which: int = 0):
        nl = _i()
        rows = (_i * 32)()
        nnz = (_i64 * 32)()
        _check(lib().sdg_precond_hierarchy(self.h, which, C.byref(nl), rows, nnz, 32))
        return [(rows[k], nnz[k]) for k in range(nl.value)]

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib is not None:
            _lib.sdg_precond_destroy(h)
            self.h = None


class IdentityPreconditioner(Preconditioner):
    def __init__(self, n: int, ctx: Optional[Context] = None):
        ctx = ctx or default_context()
        h = _vp()
        _check(lib().sdg_identity_create(ctx.h, n, C.byref(h)))
        super().__init__(h, ctx)


class Ilu0Preconditioner(Preconditioner):
    """Ilu0Preconditioner (precond.hpp:18-30, precond.cpp:13-87): the
    reference's ILU(0) factors; the two triangular solves on the device."""

    def __init__(self, a: "SparseMatrix", ctx: Optional[Context] = None):
        ctx = ctx or default_context()
        if a.n_rows != a.n_cols:
            raise ValueError("ilu0: matrix must be square")
        h = _vp()
        _check(lib().sdg_ilu0_create(a.device(ctx).h, C.byref(h)))
        super().__init__(h, ctx, [a])


@dataclass
class AmgOptions:
    max_levels: int = 3
    strength_theta: float = 0.08
    coarse_threshold: int = 100
    components: list = field(default_factory=list)

    def _c(self, n_rows: int):
        o = _AmgOpts(self.max_levels, self.strength_theta, self.coarse_threshold, None)
        keep = None
        if self.components is not None and len(self.components):
            if len(self.components) != n_rows:
                raise ValueError("amg_setup: component label length mismatch")
            keep = _i32(self.components)
            o.components = keep.ctypes.data_as(C.POINTER(_i))
        return o, keep


class AmgPreconditioner(Preconditioner):
    """Aggregation AMG V(1,1) (precond.hpp:101-120)."""

    def __init__(self, a: SparseMatrix, opts: Optional[AmgOptions] = None, ctx: Optional[Context] = None):
        ctx = ctx or default_context()
        opts = opts or AmgOptions()
        if a.n_rows != a.n_cols:
            raise ValueError("amg_setup: matrix must be square")
        o, keep = opts._c(a.n_rows)
        h = _vp()
        _check(lib().sdg_amg_create(a.device(ctx).h, C.byref(o), C.byref(h)))
        super().__init__(h, ctx, [keep])


@dataclass
class UzawaConfig:
    amg: AmgOptions = field(default_factory=AmgOptions)
    power_tol_rel: float = 1e-3
    power_max_iters: int = 200
    power_seed: int = 1729
    omega_override: float = float("nan")


class UzawaPreconditioner(Preconditioner):
    """Inexact Uzawa sweep (precond.cpp:264-299)."""

    def __init__(self, v: SparseMatrix, b: SparseMatrix, c: SparseMatrix, cfg: Optional[UzawaConfig] = None,
                 ctx: Optional[Context] = None):
        ctx = ctx or default_context()
        cfg = cfg or UzawaConfig()
        amg, keep = cfg.amg._c(v.n_rows)
        o = _UzawaOpts(amg, cfg.power_tol_rel, cfg.power_max_iters, cfg.power_seed, cfg.omega_override)
        h = _vp()
        _check(lib().sdg_uzawa_create(v.device(ctx).h, b.device(ctx).h, c.device(ctx).h, C.byref(o), C.byref(h)))
        super().__init__(h, ctx, [keep])

    def omega(self) -> float:
        return lib().sdg_precond_omega(self.h)


@dataclass
class HostLevel:
    a: SparseMatrix
    aggregate_of: Optional[np.ndarray]
    n_coarse: int
    schedule_depth: int


def host_hierarchy(a: SparseMatrix, opts: Optional[AmgOptions] = None) -> list:
    """The aggregation hierarchy the device AMG is built from (host setup only, no GPU)."""
    opts = opts or AmgOptions()
    if a.n_rows != a.n_cols:
        raise ValueError("amg_setup: matrix must be square")
    o, keep = opts._c(a.n_rows)
    h = _vp()
    L = lib()
    _check(L.sdg_host_hierarchy_build(a.n_rows, a.row_offsets, a.col_indices,
                                      a.values if a.values.size else np.zeros(1), C.byref(o), C.byref(h)))
    try:
        out = []
        nl = L.sdg_host_hierarchy_levels(h)
        for lev in range(nl):
            n, nnz, nc, sd = _i(), _i64(), _i(), _i()
            _check(L.sdg_host_hierarchy_level(h, lev, C.byref(n), C.byref(nnz), C.byref(nc), C.byref(sd),
                                              None, None, None, None))
            rp = np.empty(n.value + 1, np.int32)
            ci = np.empty(max(nnz.value, 1), np.int32)
            vv = np.empty(max(nnz.value, 1), np.float64)
            agg = np.empty(max(n.value, 1), np.int32) if lev + 1 < nl else None
            _check(L.sdg_host_hierarchy_level(h, lev, None, None, None, None, rp.ctypes.data_as(_vp),
                                              ci.ctypes.data_as(_vp), vv.ctypes.data_as(_vp),
                                              None if agg is None else agg.ctypes.data_as(_vp)))
            out.append(HostLevel(SparseMatrix(n.value, n.value, rp, ci[:nnz.value], vv[:nnz.value]),
                                 None if agg is None else agg[:n.value], nc.value, sd.value))
        return out
    finally:
        L.sdg_host_hierarchy_destroy(h)
        del keep


class BlockPrecondKind(IntEnum):
    td_bj = 0
    td_bgs = 1
    pv_bj = 2
    pv_bgs = 3


class BlockPreconditioner(Preconditioner):
    """precond.cpp:304-363."""

    def __init__(self, kind: BlockPrecondKind, matrix: SparseMatrix, n_v: int, n_pff: int, n_ppm: int,
                 first: Optional[Preconditioner], pm: Optional[Preconditioner], ctx: Optional[Context] = None):
        ctx = ctx or default_context()
        h = _vp()
        _check(lib().sdg_block_create(int(kind), matrix.device(ctx).h, n_v, n_pff, n_ppm,
                                      first.h if first else None, pm.h if pm else None, C.byref(h)))
        super().__init__(h, ctx, [first, pm])
        self.kind = BlockPrecondKind(kind)

    def omega(self) -> float:
        return lib().sdg_precond_omega(self.h)


class TdPreconditioner(Preconditioner):
    """MonolithicDriver::build_preconditioner (bench.cpp:121-182) for td_bj /
    td_bgs(Uzawa(AMG_V), AMG_D') in one setup call."""

    def __init__(self, system: "CoupledSystem", kind: str = "td_bgs", v_max_levels: int = 3,
                 d_max_levels: int = 3, omega_override: float = float("nan"), ctx: Optional[Context] = None):
        ctx = ctx or default_context()
        k = {"td_bj": 0, "td_bgs": 1, "td_bj_ilu0": 0 | 16, "td_bgs_ilu0": 1 | 16}[kind]  # SDG_TD_ILU0
        h = _vp()
        s = system
        _check(lib().sdg_td_create(s.matrix.device(ctx).h, s.n_u, s.n_vel, s.n_pff, s.n_ppm, k, v_max_levels,
                                   d_max_levels, omega_override, C.byref(h)))
        super().__init__(h, ctx)
        self.kind = kind

    def omega(self) -> float:
        return lib().sdg_precond_omega(self.h)


# ---------------------------------------------------------------------------
# Krylov


@dataclass
class RestartController:
    """krylov.hpp:23-47 (the reference passes it by value)."""
    m_init: int = 3
    m_min: int = 3
    m_step: int = 5
    m_max: int = 53
    current_m: int = 3
    previous_rate: float = 0.0
    has_rate_sample: bool = False
    alpha_p: float = -3.0
    alpha_d: float = 5.0
    stall_threshold: float = 0.05

    @staticmethod
    def defaults() -> "RestartController":
        return RestartController()

    @staticmethod
    def fixed(m: int) -> "RestartController":
        """GMRES(m): m_init = m_min = m_max = current_m = m."""
        return RestartController(m_init=m, m_min=m, m_max=m, current_m=m)

    def reset(self):
        self.current_m = self.m_init
        self.previous_rate = 0.0
        self.has_rate_sample = False

    def update(self, rate: float):
        """krylov.cpp:37-45 (host-side, for tests of the rule itself)."""
        rate = min(max(rate, -16.0), 16.0)
        derivative = (rate - self.previous_rate) if self.has_rate_sample else 0.0
        delta = int(math.floor(self.alpha_p * rate + self.alpha_d * derivative))
        if rate > -self.stall_threshold:
            delta = max(delta, self.m_step)
        self.current_m = min(max(self.current_m + delta, self.m_min), self.m_max)
        self.previous_rate = rate
        self.has_rate_sample = True

    def _c(self) -> _Restart:
        return _Restart(self.m_init, self.m_min, self.m_step, self.m_max, self.current_m, self.previous_rate,
                        int(self.has_rate_sample), self.alpha_p, self.alpha_d, self.stall_threshold)


@dataclass
class SolveReport:
    iterations: int = 0
    residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    converged: bool = False
    wall_time: float = 0.0
    final_residual: float = 0.0
    precond_applications: int = 0
    device_ms: float = 0.0
    breakdown: bool = False  # warm-started BiCGSTAB ended by a repeated breakdown


@dataclass
class GmresResult:
    x: np.ndarray
    report: SolveReport


def _report(rep: _Report, hist: np.ndarray) -> SolveReport:
    n = min(rep.history_length, hist.size)
    return SolveReport(rep.iterations, hist[:n].copy(), bool(rep.converged), rep.wall_time, rep.final_residual,
                       rep.precond_applications, rep.device_ms, bool(rep.breakdown))


def _operator_matrix(op) -> SparseMatrix:
    if isinstance(op, SparseMatrix):
        return op
    if isinstance(op, LinearOperator) and op.matrix is not None:
        return op.matrix
    raise TypeError("the device solvers need a matrix-backed LinearOperator (LinearOperator.from_matrix)")


def pd_gmres(op, precond: Optional[Preconditioner], b, tol_abs: float, max_restarts: int,
             ctrl: Optional[RestartController] = None, history_capacity: int = 1 << 16) -> GmresResult:
    """Right-preconditioned restarted GMRES (krylov.cpp:47-184) on the GPU."""
    a = _operator_matrix(op)
    b = _f64(b)
    if b.size != a.n_rows:
        raise ValueError("pd_gmres: dimension mismatch")
    ctrl = ctrl or RestartController.defaults()
    ctx = precond.ctx if precond is not None else default_context()
    x = np.empty(a.n_rows)
    hist = np.empty(history_capacity)
    rep = _Report()
    rep.residual_history = hist.ctypes.data_as(C.POINTER(_d))
    rep.history_capacity = history_capacity
    rc = _c = ctrl._c()
    _check(lib().sdg_pd_gmres(a.device(ctx).h, precond.h if precond else None, b, x, tol_abs, max_restarts,
                              C.byref(rc), C.byref(rep)))
    del _c
    return GmresResult(x, _report(rep, hist))


def pd_gmres_warm(op, precond: Optional[Preconditioner], b, x0, tol_abs: float, max_restarts: int,
                  ctrl: Optional[RestartController] = None, history_capacity: int = 1 << 16) -> GmresResult:
    """Warm-started pd_gmres: the reference solve (x0 = 0, krylov.cpp:58) of the
    correction d in A d = b - A x0, returning x0 + d (BASELINE config 4)."""
    a = _operator_matrix(op)
    b = _f64(b)
    x = _f64(x0).copy()
    if b.size != a.n_rows or x.size != a.n_rows:
        raise ValueError("pd_gmres: dimension mismatch")
    ctrl = ctrl or RestartController.defaults()
    ctx = precond.ctx if precond is not None else default_context()
    hist = np.empty(history_capacity)
    rep = _Report()
    rep.residual_history = hist.ctypes.data_as(C.POINTER(_d))
    rep.history_capacity = history_capacity
    rc = ctrl._c()
    _check(lib().sdg_pd_gmres_warm(a.device(ctx).h, precond.h if precond else None, b, x, tol_abs, max_restarts,
                                   C.byref(rc), C.byref(rep)))
    return GmresResult(x, _report(rep, hist))


def bicgstab_warm(op, precond: Optional[Preconditioner], b, x0, tol_abs: float, max_iters: int,
                  history_capacity: int = 1 << 16) -> GmresResult:
    """Warm-started bicgstab: the reference solve (x0 = 0, krylov.cpp:194) of the
    correction d in A d = b - A x0, returning x0 + d."""
    a = _operator_matrix(op)
    b = _f64(b)
    x = _f64(x0).copy()
    if b.size != a.n_rows or x.size != a.n_rows:
        raise ValueError("bicgstab: dimension mismatch")
    ctx = precond.ctx if precond is not None else default_context()
    hist = np.empty(history_capacity)
    rep = _Report()
    rep.residual_history = hist.ctypes.data_as(C.POINTER(_d))
    rep.history_capacity = history_capacity
    _check(lib().sdg_bicgstab_warm(a.device(ctx).h, precond.h if precond else None, b, x, tol_abs, max_iters,
                                   C.byref(rep)))
    return GmresResult(x, _report(rep, hist))


def bicgstab(op, precond: Optional[Preconditioner], b, tol_abs: float, max_iters: int,
             history_capacity: int = 1 << 16) -> GmresResult:
    """Right-preconditioned BiCGSTAB (krylov.cpp:186-292) on the GPU."""
    a = _operator_matrix(op)
    b = _f64(b)
    if b.size != a.n_rows:
        raise ValueError("bicgstab: dimension mismatch")
    ctx = precond.ctx if precond is not None else default_context()
    x = np.empty(a.n_rows)
    hist = np.empty(history_capacity)
    rep = _Report()
    rep.residual_history = hist.ctypes.data_as(C.POINTER(_d))
    rep.history_capacity = history_capacity
    _check(lib().sdg_bicgstab(a.device(ctx).h, precond.h if precond else None, b, x, tol_abs, max_iters,
                              C.byref(rep)))
    return GmresResult(x, _report(rep, hist))


@dataclass
class PowerIterationResult:
    value: float = 0.0
    converged: bool = False
    iterations: int = 0


def power_iteration(op, tol_rel: float, max_iters: int, seed: int) -> PowerIterationResult:
    """krylov.cpp:307-339 on y = A x (device)."""
    a = _operator_matrix(op)
    v, it, cv = _d(), _i(), _i()
    _check(lib().sdg_power_iteration(a.device().h, tol_rel, max_iters, seed, C.byref(v), C.byref(it), C.byref(cv)))
    return PowerIterationResult(v.value, bool(cv.value), it.value)


# ---------------------------------------------------------------------------
# assembly (host C++ inside libsdgpu.so)


@dataclass
class ScenarioConfig:
    """config.hpp:38-58 fields used by assemble_monolithic; n x n free-flow box."""
    cells_per_unit_square: int = 16
    permeability: float = 1e-6
    alpha_bj: float = 1.0
    kinematic_viscosity: float = 1e-6
    density: float = 1000.0
    dt: float = 2e5
    t_end: float = 50e5
    dp_max: float = 1e-9

    def dynamic_viscosity(self) -> float:
        return self.kinematic_viscosity * self.density

    def inflow_pressure(self, t: float) -> float:
        return self.dp_max * 0.5 * (1.0 - math.cos(math.pi * t / self.t_end))


@dataclass
class CoupledSystem:
    """assembly.hpp:95-106 (matrix, rhs and the [v | p_ff | p_pm] ranges)."""
    matrix: SparseMatrix
    rhs: np.ndarray
    n: int
    n_u: int
    n_vel: int
    n_pff: int
    n_ppm: int

    @property
    def n_ff(self) -> int:
        return self.n_vel + self.n_pff

    def n_total(self) -> int:
        return self.matrix.n_rows


def assemble_monolithic(cfg: ScenarioConfig, t: Optional[float] = None, v_prev=None, k_cell=None) -> CoupledSystem:
    """assemble_monolithic (assembly.cpp:327-380) on the n x n free-flow box.

    ``k_cell`` (n*n, row-major) switches on the per-cell permeability
    extension (BASELINE.json configs 2/4); None reproduces the reference
    bitwise.
    """
    n = cfg.cells_per_unit_square
    sc = _Scenario(n, cfg.permeability, cfg.alpha_bj, cfg.kinematic_viscosity, cfg.density, cfg.dt, cfg.t_end,
                   cfg.dp_max, cfg.t_end if t is None else t)
    kc = None if k_cell is None else _f64(k_cell)
    vp = None if v_prev is None else _f64(v_prev)
    if kc is not None and kc.size != n * n:
        raise ValueError("assemble_monolithic: k_cell must have n*n entries")
    kcp = None if kc is None else kc.ctypes.data_as(_vp)
    vpp = None if vp is None else vp.ctypes.data_as(_vp)
    N, nu, nv, npf, npm = _i(), _i(), _i(), _i(), _i()
    nnz = _i64()
    L = lib()
    _check(L.sdg_assemble_monolithic(C.byref(sc), kcp, vpp, C.byref(N), C.byref(nnz), C.byref(nu), C.byref(nv),
                                     C.byref(npf), C.byref(npm), None, None, None, None))
    rp = np.empty(N.value + 1, np.int32)
    ci = np.empty(nnz.value, np.int32)
    vv = np.empty(nnz.value, np.float64)
    rhs = np.empty(N.value, np.float64)
    _check(L.sdg_assemble_monolithic(C.byref(sc), kcp, vpp, None, None, None, None, None, None,
                                     rp.ctypes.data_as(_vp), ci.ctypes.data_as(_vp), vv.ctypes.data_as(_vp),
                                     rhs.ctypes.data_as(_vp)))
    return CoupledSystem(SparseMatrix(N.value, N.value, rp, ci, vv), rhs, n, nu.value, nv.value, npf.value,
                         npm.value)


def assemble_rhs_device(cfg: ScenarioConfig, rhs_ptr: int, v_prev_ptr: Optional[int] = None,
                        t: Optional[float] = None, ctx: Optional[Context] = None) -> None:
    """The right-hand side of assemble_monolithic on the device (stream-ordered on
    the context's stream), from the previous velocity at device address
    ``v_prev_ptr`` (None: zero); bitwise the host assembly's rhs."""
    ctx = ctx or default_context()
    sc = _scenario_c(cfg, t)
    _check(lib().sdg_assemble_rhs_device(ctx.h, C.byref(sc), None if v_prev_ptr is None else C.c_void_p(v_prev_ptr),
                                         C.c_void_p(rhs_ptr)))


def assemble_matrix_device(cfg: ScenarioConfig, k_cell=None, t: Optional[float] = None,
                           ctx: Optional[Context] = None) -> SparseMatrix:
    """The matrix of assemble_monolithic assembled on the device (sdg_assemble_matrix_device:
    count pass, device scan, fill pass) and copied back as a SparseMatrix; bitwise the
    host assembly, per-cell permeability included."""
    import torch
    ctx = ctx or default_context()
    sc = _scenario_c(cfg, t)
    n = cfg.cells_per_unit_square
    n_total = 2 * n * (n + 1) + 2 * n * n
    dev = torch.device("cuda")
    kd = None if k_cell is None else torch.from_numpy(np.ascontiguousarray(k_cell, dtype=np.float64)).to(dev)
    rp = torch.empty(n_total + 1, dtype=torch.int32, device=dev)
    nnz = _i64()
    kp = None if kd is None else C.c_void_p(kd.data_ptr())
    _check(lib().sdg_assemble_matrix_device(ctx.h, C.byref(sc), kp, C.c_void_p(rp.data_ptr()), None, None, 0,
                                            C.byref(nnz)))
    ci = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=dev)
    vv = torch.empty(max(nnz.value, 1), dtype=torch.float64, device=dev)
    _check(lib().sdg_assemble_matrix_device(ctx.h, C.byref(sc), kp, C.c_void_p(rp.data_ptr()),
                                            C.c_void_p(ci.data_ptr()), C.c_void_p(vv.data_ptr()), nnz.value,
                                            C.byref(nnz)))
    return SparseMatrix(n_total, n_total, rp.cpu().numpy(), ci.cpu().numpy()[:nnz.value],
                        vv.cpu().numpy()[:nnz.value])


def _scenario_c(cfg: "ScenarioConfig", t: Optional[float]) -> _Scenario:
    return _Scenario(cfg.cells_per_unit_square, cfg.permeability, cfg.alpha_bj, cfg.kinematic_viscosity,
                     cfg.density, cfg.dt, cfg.t_end, cfg.dp_max, cfg.t_end if t is None else t)


def _two_phase(call):
    n, nnz = _i(), _i64()
    _check(call(C.byref(n), C.byref(nnz), None, None, None, None))
    rp = np.empty(n.value + 1, np.int32)
    ci = np.empty(nnz.value, np.int32)
    vv = np.empty(nnz.value, np.float64)
    rhs = np.empty(n.value, np.float64)
    _check(call(None, None, rp.ctypes.data_as(_vp), ci.ctypes.data_as(_vp), vv.ctypes.data_as(_vp),
                rhs.ctypes.data_as(_vp)))
    return SparseMatrix(n.value, n.value, rp, ci, vv), rhs


def assemble_stokes(cfg: "ScenarioConfig", v_gamma, t: Optional[float] = None, v_prev=None):
    """assemble_stokes (assembly.cpp:287-303) on the n x n free-flow box with
    Dirichlet interface velocities v_gamma (the partitioned driver's free-flow
    problem, coupling.cpp:218-229).  Returns (matrix, rhs)."""
    sc = _scenario_c(cfg, t)
    vg = _f64(v_gamma)
    if vg.size != cfg.cells_per_unit_square:
        raise ValueError("assemble_stokes: interface data length mismatch")
    vp = None if v_prev is None else _f64(v_prev)
    vpp = None if vp is None else vp.ctypes.data_as(_vp)
    return _two_phase(lambda n, nnz, rp, ci, vv, rhs: lib().sdg_assemble_stokes(
        C.byref(sc), vpp, vg.ctypes.data_as(_vp), n, nnz, rp, ci, vv, rhs))


def assemble_darcy(cfg: "ScenarioConfig", p_gamma):
    """assemble_darcy (assembly.cpp:305-325) on the n x n porous box with
    Dirichlet interface pressures p_gamma (coupling.cpp:231-242)."""
    sc = _scenario_c(cfg, None)
    pg = _f64(p_gamma)
    if pg.size != cfg.cells_per_unit_square:
        raise ValueError("assemble_darcy: interface data length mismatch")
    return _two_phase(lambda n, nnz, rp, ci, vv, rhs: lib().sdg_assemble_darcy(
        C.byref(sc), pg.ctypes.data_as(_vp), n, nnz, rp, ci, vv, rhs))


def stokes_pressure_trace(cfg: "ScenarioConfig", x_ff) -> np.ndarray:
    out = np.empty(cfg.cells_per_unit_square)
    _check(lib().sdg_stokes_pressure_trace(C.byref(_scenario_c(cfg, None)), _f64(x_ff), out))
    return out


def darcy_velocity_trace(cfg: "ScenarioConfig", p, p_gamma) -> np.ndarray:
    out = np.empty(cfg.cells_per_unit_square)
    _check(lib().sdg_darcy_velocity_trace(C.byref(_scenario_c(cfg, None)), _f64(p), _f64(p_gamma), out))
    return out


# ---------------------------------------------------------------------------
# device-pointer entry points (inputs already resident in HBM)


def _solve_device(fn, a: SparseMatrix, precond, b_ptr: int, x_ptr: int, *args, ctx=None,
                  history_capacity: int = 1 << 16):
    ctx = ctx or (precond.ctx if precond is not None else default_context())
    hist = np.empty(history_capacity)
    rep = _Report()
    rep.residual_history = hist.ctypes.data_as(C.POINTER(_d))
    rep.history_capacity = history_capacity
    _check(fn(a.device(ctx).h, precond.h if precond else None, _vp(b_ptr), _vp(x_ptr), *args, C.byref(rep)))
    return _report(rep, hist)


def bicgstab_device(a: SparseMatrix, precond: Optional[Preconditioner], b_ptr: int, x_ptr: int, tol_abs: float,
                    max_iters: int, ctx: Optional[Context] = None) -> SolveReport:
    """sdg_bicgstab_device: b and x are device pointers on the context's device."""
    return _solve_device(lib().sdg_bicgstab_device, a, precond, b_ptr, x_ptr, tol_abs, max_iters, ctx=ctx)


def bicgstab_warm_device(a: SparseMatrix, precond: Optional[Preconditioner], b_ptr: int, x_ptr: int,
                         tol_abs: float, max_iters: int, ctx: Optional[Context] = None) -> SolveReport:
    return _solve_device(lib().sdg_bicgstab_warm_device, a, precond, b_ptr, x_ptr, tol_abs, max_iters, ctx=ctx)


def pd_gmres_warm_device(a: SparseMatrix, precond: Optional[Preconditioner], b_ptr: int, x_ptr: int,
                         tol_abs: float, max_restarts: int, ctrl: Optional[RestartController] = None,
                         ctx: Optional[Context] = None) -> SolveReport:
    rc = (ctrl or RestartController.defaults())._c()
    return _solve_device(lib().sdg_pd_gmres_warm_device, a, precond, b_ptr, x_ptr, tol_abs, max_restarts,
                         C.byref(rc), ctx=ctx)


def pd_gmres_device(a: SparseMatrix, precond: Optional[Preconditioner], b_ptr: int, x_ptr: int, tol_abs: float,
                    max_restarts: int, ctrl: Optional[RestartController] = None,
                    ctx: Optional[Context] = None) -> SolveReport:
    rc = (ctrl or RestartController.defaults())._c()
    return _solve_device(lib().sdg_pd_gmres_device, a, precond, b_ptr, x_ptr, tol_abs, max_restarts, C.byref(rc),
                         ctx=ctx)
