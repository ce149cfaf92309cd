"""ORACLE / TEST INFRASTRUCTURE ONLY -- ctypes view of the checker libraries.

* ``RefLib``  -> ``oracle/_ref/libsdcore_ref.so``: the UNMODIFIED reference
  library (``/root/reference/proj/core/src``) plus the C-ABI shim
  ``oracle/ref_harness.cpp``.
* ``PortLib`` -> ``oracle/_ref/liboracle_port.so``: the plain-C restatement of
  the hot path (``oracle/sdc_oracle.c``), pinned against ``RefLib``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsdcore_ref.so")
PORT_SO = os.path.join(HERE, "_ref", "liboracle_port.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_vp = C.c_void_p
_i = C.c_int
_d = C.c_double


def _f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def _i32(x):
    return np.ascontiguousarray(x, dtype=np.int32)


@dataclass
class Csr:
    n_rows: int
    n_cols: int
    rowptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.n_rows, self.n_cols))
        for i in range(self.n_rows):
            s, e = self.rowptr[i], self.rowptr[i + 1]
            d[i, self.col[s:e]] += self.val[s:e]
        return d

    @staticmethod
    def from_dense(d: np.ndarray) -> "Csr":
        d = np.asarray(d, dtype=np.float64)
        rp = [0]
        ci, vv = [], []
        for i in range(d.shape[0]):
            nz = np.nonzero(d[i])[0]
            ci.extend(nz.tolist())
            vv.extend(d[i, nz].tolist())
            rp.append(len(ci))
        return Csr(d.shape[0], d.shape[1], _i32(rp), _i32(ci), _f64(vv))


@dataclass
class System:
    n: int
    n_u: int
    n_vel: int
    n_pff: int
    n_ppm: int
    a: Csr
    rhs: np.ndarray

    @property
    def n_ff(self) -> int:
        return self.n_vel + self.n_pff


@dataclass
class SolveReport:
    iterations: int
    final_residual: float
    converged: bool
    wall_time: float
    residual_history: np.ndarray = field(repr=False)


@dataclass
class Level:
    a: Csr
    aggregate_of: np.ndarray | None
    n_coarse: int


def _proto(lib, name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


class RefLib:
    """The reference library itself (checker + CPU baseline)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref`")
        L = C.CDLL(path)
        self.L = L
        p = lambda n, r, a: _proto(L, n, r, a)  # noqa: E731
        p("ref_last_error", C.c_char_p, [])
        p("ref_system_new", _i, [_i, _d, _d, _d, _d, _d, _d, _d, _d, _vp, C.POINTER(_vp)])
        p("ref_system_sizes", None, [_vp] + [C.POINTER(_i), C.POINTER(C.c_longlong)] + [C.POINTER(_i)] * 4)
        p("ref_system_copy", None, [_vp, _ip, _ip, _dp, _dp])
        p("ref_system_free", None, [_vp])
        p("ref_system_traces", _i, [_vp, _dp, _dp, _dp])
        p("ref_spmv", _i, [_i, _i, _ip, _ip, _dp, _dp, _dp])
        p("ref_spmv_add", _i, [_i, _i, _ip, _ip, _dp, _dp, _dp, _d])
        p("ref_sor_sweep", _i, [_i, _ip, _ip, _dp, _dp, _dp, _d])
        p("ref_random_vector", None, [_i, C.c_uint, _dp])
        p("ref_random_dominant", _i, [_i, _d, C.c_uint, _i, C.POINTER(_vp)])
        p("ref_matrix_new", _i, [_i, _i, _ip, _ip, _dp, C.POINTER(_vp)])
        p("ref_matrix_sizes", None, [_vp, C.POINTER(_i), C.POINTER(_i), C.POINTER(C.c_longlong)])
        p("ref_matrix_copy", None, [_vp, _ip, _ip, _dp])
        p("ref_matrix_free", None, [_vp])
        p("ref_stokes_new", _i, [_i, _d, _d, _d, _d, _d, _d, _d, _d, _vp, _dp, C.POINTER(_vp), _dp])
        p("ref_darcy_new", _i, [_i, _d, _dp, C.POINTER(_vp), _dp])
        p("ref_stokes_pressure_trace", _i, [_i, _d, _dp, _dp])
        p("ref_darcy_velocity_trace", _i, [_i, _d, _dp, _dp, _dp])
        p("ref_uzawa_stokes_new", _i, [_vp, _i, _i, C.POINTER(_vp)])
        p("ref_amg_precond_new", _i, [_vp, _i, C.POINTER(_vp)])
        p("ref_precond_free", None, [_vp])
        p("ref_ilu0_new", _i, [_vp, C.POINTER(_vp)])
        p("ref_precond_apply", _i, [_vp, _dp, _dp])
        p("ref_ground_dof", _i, [_vp, _i, C.POINTER(_vp)])
        p("ref_amg_setup", _i, [_vp, _i, _d, _i, _vp, C.POINTER(_vp)])
        p("ref_hier_num_levels", _i, [_vp])
        p("ref_hier_level_sizes", None, [_vp, _i, C.POINTER(_i), C.POINTER(C.c_longlong), C.POINTER(_i)])
        p("ref_hier_level_copy", None, [_vp, _i, _ip, _ip, _dp, _vp])
        p("ref_hier_coarse_lu_sizes", None, [_vp, C.POINTER(_i), C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)])
        p("ref_hier_coarse_lu_copy", None, [_vp, _ip, _ip, _dp, _ip, _ip, _dp, _ip])
        p("ref_hier_vcycle", _i, [_vp, _dp, _dp])
        p("ref_hier_free", None, [_vp])
        p("ref_lu_solve_dense_check", _i, [_vp, _dp, _dp])
        p("ref_td_new", _i, [_i, _ip, _ip, _dp, _i, _i, _i, _i, _i, _i, _i, C.POINTER(_vp)])
        p("ref_td_omega", _d, [_vp])
        p("ref_td_setup_seconds", _d, [_vp])
        p("ref_td_v_hier", _vp, [_vp])
        p("ref_td_d_hier", _vp, [_vp])
        p("ref_td_apply", _i, [_vp, _dp, _dp])
        p("ref_uzawa_apply", _i, [_vp, _dp, _dp])
        p("ref_td_free", None, [_vp])
        rep = [C.POINTER(_i), C.POINTER(_d), C.POINTER(_i), C.POINTER(_d), _dp, _i, C.POINTER(_i)]
        p("ref_pd_gmres", _i, [_vp, _i, _vp, _dp, _d, _i, _i, _i, _i, _i, _dp] + rep)
        p("ref_bicgstab", _i, [_vp, _i, _vp, _dp, _d, _i, _dp] + rep)
        p("ref_power_iteration", _i, [_vp, _d, _i, C.c_uint, C.POINTER(_d), C.POINTER(_i), C.POINTER(_i)])

    # -- errors ------------------------------------------------------------
    def _check(self, rc: int):
        if rc == 0:
            return
        msg = self.L.ref_last_error().decode()
        if rc == 1:
            raise ValueError(msg)
        raise RuntimeError(msg)

    # -- assembly ----------------------------------------------------------
    def assemble(self, n, permeability=1.0, alpha_bj=1.0, nu=1.0, rho=1.0, dt=float("inf"),
                 t_end=1.0, dp_max=1.0, t=None, v_prev=None) -> System:
        """Reference ``assemble_monolithic`` on the n x n free-flow box."""
        if t is None:
            t = t_end
        h = _vp()
        vp = None if v_prev is None else _f64(v_prev).ctypes.data_as(_vp)
        self._check(self.L.ref_system_new(n, permeability, alpha_bj, nu, rho, dt, t_end, dp_max, t, vp, C.byref(h)))
        try:
            nn, nu_, nv, npf, npm = _i(), _i(), _i(), _i(), _i()
            nnz = C.c_longlong()
            self.L.ref_system_sizes(h, C.byref(nn), C.byref(nnz), C.byref(nu_), C.byref(nv), C.byref(npf), C.byref(npm))
            rp = np.empty(nn.value + 1, np.int32)
            ci = np.empty(nnz.value, np.int32)
            vv = np.empty(nnz.value, np.float64)
            rhs = np.empty(nn.value, np.float64)
            self.L.ref_system_copy(h, rp, ci, vv, rhs)
        finally:
            self.L.ref_system_free(h)
        return System(nn.value, nu_.value, nv.value, npf.value, npm.value,
                      Csr(nn.value, nn.value, rp, ci, vv), rhs)

    # -- kernels -----------------------------------------------------------
    def spmv(self, a: Csr, x):
        y = np.empty(a.n_rows)
        self._check(self.L.ref_spmv(a.n_rows, a.n_cols, a.rowptr, a.col, a.val, _f64(x), y))
        return y

    def spmv_add(self, a: Csr, x, y, alpha=1.0):
        y = _f64(y).copy()
        self._check(self.L.ref_spmv_add(a.n_rows, a.n_cols, a.rowptr, a.col, a.val, _f64(x), y, alpha))
        return y

    def sor_sweep(self, a: Csr, z, r, omega=1.0):
        z = _f64(z).copy()
        self._check(self.L.ref_sor_sweep(a.n_rows, a.rowptr, a.col, a.val, z, _f64(r), omega))
        return z

    def random_vector(self, n, seed):
        out = np.empty(n)
        self.L.ref_random_vector(n, seed, out)
        return out

    def random_dominant(self, n, density, seed, symmetric=False) -> Csr:
        h = _vp()
        self._check(self.L.ref_random_dominant(n, density, seed, int(symmetric), C.byref(h)))
        try:
            return self._matrix_copy(h)
        finally:
            self.L.ref_matrix_free(h)

    def _matrix_copy(self, h) -> Csr:
        r, c = _i(), _i()
        nnz = C.c_longlong()
        self.L.ref_matrix_sizes(h, C.byref(r), C.byref(c), C.byref(nnz))
        rp = np.empty(r.value + 1, np.int32)
        ci = np.empty(nnz.value, np.int32)
        vv = np.empty(nnz.value, np.float64)
        self.L.ref_matrix_copy(h, rp, ci, vv)
        return Csr(r.value, c.value, rp, ci, vv)

    def matrix(self, a: Csr) -> "RefMatrix":
        return RefMatrix(self, a)

    # -- partitioned pieces (coupling.cpp:218-242) --------------------------
    def stokes(self, n, permeability=1.0, alpha_bj=1.0, nu=1.0, rho=1.0, dt=float("inf"), t_end=1.0, dp_max=1.0,
               t=None, v_prev=None, v_gamma=None):
        """Reference assemble_stokes on the n x n box with Dirichlet interface velocities v_gamma."""
        t = t_end if t is None else t
        nt = 2 * n * (n + 1) + n * n
        rhs = np.empty(nt)
        h = _vp()
        vp = None if v_prev is None else _f64(v_prev).ctypes.data_as(_vp)
        self._check(self.L.ref_stokes_new(n, permeability, alpha_bj, nu, rho, dt, t_end, dp_max, t, vp,
                                          _f64(v_gamma), C.byref(h), rhs))
        try:
            return self._matrix_copy(h), rhs
        finally:
            self.L.ref_matrix_free(h)

    def darcy(self, n, k_over_mu, p_gamma):
        """Reference assemble_darcy on the n x n box with Dirichlet interface pressures p_gamma."""
        rhs = np.empty(n * n)
        h = _vp()
        self._check(self.L.ref_darcy_new(n, k_over_mu, _f64(p_gamma), C.byref(h), rhs))
        try:
            return self._matrix_copy(h), rhs
        finally:
            self.L.ref_matrix_free(h)

    def stokes_pressure_trace(self, n, mu, x):
        out = np.empty(n)
        self._check(self.L.ref_stokes_pressure_trace(n, mu, _f64(x), out))
        return out

    def darcy_velocity_trace(self, n, k_over_mu, p, p_gamma):
        out = np.empty(n)
        self._check(self.L.ref_darcy_velocity_trace(n, k_over_mu, _f64(p), _f64(p_gamma), out))
        return out

    def uzawa_stokes(self, a: Csr, n, max_levels=3) -> "RefPrecond":
        with self.matrix(a) as m:
            h = _vp()
            self._check(self.L.ref_uzawa_stokes_new(m.h, n, max_levels, C.byref(h)))
            return RefPrecond(self, h)

    def amg_precond(self, a: Csr, max_levels=3) -> "RefPrecond":
        with self.matrix(a) as m:
            h = _vp()
            self._check(self.L.ref_amg_precond_new(m.h, max_levels, C.byref(h)))
            return RefPrecond(self, h)

    def ilu0(self, a: Csr) -> "RefPrecond":
        """Ilu0Preconditioner (precond.cpp:13-87)."""
        with self.matrix(a) as m:
            h = _vp()
            self._check(self.L.ref_ilu0_new(m.h, C.byref(h)))
            return RefPrecond(self, h)

    def precond_apply(self, p: "RefPrecond", r):
        z = np.empty(len(r))
        self._check(self.L.ref_precond_apply(p.h, _f64(r), z))
        return z

    def ground_dof(self, a: Csr, dof=0) -> Csr:
        with self.matrix(a) as m:
            h = _vp()
            self._check(self.L.ref_ground_dof(m.h, dof, C.byref(h)))
            try:
                return self._matrix_copy(h)
            finally:
                self.L.ref_matrix_free(h)

    # -- AMG ---------------------------------------------------------------
    def amg_setup(self, a: Csr, max_levels=3, theta=0.08, coarse_threshold=100, components=None) -> "RefHierarchy":
        with self.matrix(a) as m:
            h = _vp()
            comp = None if components is None else _i32(components)
            self._check(self.L.ref_amg_setup(m.h, max_levels, theta, coarse_threshold,
                                             None if comp is None else comp.ctypes.data_as(_vp), C.byref(h)))
            return RefHierarchy(self, h, owned=True, keep=comp)

    def td(self, sysm: System, kind="td_bgs", v_max_levels=3, d_max_levels=3) -> "RefTd":
        return RefTd(self, sysm, kind, v_max_levels, d_max_levels)

    def lu_solve(self, a: Csr, b):
        x = np.empty(a.n_rows)
        with self.matrix(a) as m:
            self._check(self.L.ref_lu_solve_dense_check(m.h, _f64(b), x))
        return x

    # -- solvers -----------------------------------------------------------
    def _precond_args(self, precond):
        if precond is None:
            return 0, None
        if isinstance(precond, RefTd):
            return 1, precond.h
        if isinstance(precond, RefHierarchy):
            return 2, precond.h
        if isinstance(precond, RefPrecond):
            return 3, precond.h
        raise TypeError(precond)

    def pd_gmres(self, a, b, tol_abs, max_restarts, precond=None, m_init=3, m_min=3,
                 m_step=5, m_max=53, hist_cap=1 << 16):
        """`a`: a Csr (copied into a reference SparseMatrix for the call) or a
        RefMatrix handle (borrowed, as LinearOperator::from_matrix does)."""
        kind, ph = self._precond_args(precond)
        x = np.empty(a.n_rows)
        it, fr, cv, wt, hl = _i(), _d(), _i(), _d(), _i()
        hist = np.empty(hist_cap)
        with self._borrow(a) as m:
            self._check(self.L.ref_pd_gmres(m.h, kind, ph, _f64(b), tol_abs, max_restarts, m_init, m_min,
                                            m_step, m_max, x, C.byref(it), C.byref(fr), C.byref(cv),
                                            C.byref(wt), hist, hist_cap, C.byref(hl)))
        return x, SolveReport(it.value, fr.value, bool(cv.value), wt.value, hist[: min(hl.value, hist_cap)].copy())

    def bicgstab(self, a, b, tol_abs, max_iters, precond=None, hist_cap=1 << 16):
        kind, ph = self._precond_args(precond)
        x = np.empty(a.n_rows)
        it, fr, cv, wt, hl = _i(), _d(), _i(), _d(), _i()
        hist = np.empty(hist_cap)
        with self._borrow(a) as m:
            self._check(self.L.ref_bicgstab(m.h, kind, ph, _f64(b), tol_abs, max_iters, x, C.byref(it),
                                            C.byref(fr), C.byref(cv), C.byref(wt), hist, hist_cap, C.byref(hl)))
        return x, SolveReport(it.value, fr.value, bool(cv.value), wt.value, hist[: min(hl.value, hist_cap)].copy())

    def _borrow(self, a):
        if isinstance(a, RefMatrix):
            import contextlib
            return contextlib.nullcontext(a)
        return self.matrix(a)

    def power_iteration(self, a: Csr, tol_rel, max_iters, seed):
        v, it, cv = _d(), _i(), _i()
        with self.matrix(a) as m:
            self._check(self.L.ref_power_iteration(m.h, tol_rel, max_iters, seed, C.byref(v), C.byref(it), C.byref(cv)))
        return v.value, it.value, bool(cv.value)


class RefMatrix:
    def __init__(self, lib: RefLib, a: Csr):
        self.lib = lib
        self.a = a
        self.h = _vp()
        lib._check(lib.L.ref_matrix_new(a.n_rows, a.n_cols, _i32(a.rowptr), _i32(a.col), _f64(a.val), C.byref(self.h)))

    @property
    def n_rows(self) -> int:
        return self.a.n_rows

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def close(self):
        if self.h:
            self.lib.L.ref_matrix_free(self.h)
        self.h = None


class RefPrecond:
    """An owned reference Preconditioner (Uzawa on a Stokes matrix, AMG on a Darcy matrix)."""

    def __init__(self, lib: RefLib, h):
        self.lib, self.h = lib, h

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.L.ref_precond_free(self.h)


class RefHierarchy:
    def __init__(self, lib: RefLib, h, owned: bool, keep=None, parent=None):
        self.lib, self.h, self.owned, self._keep, self._parent = lib, h, owned, keep, parent

    def __del__(self):
        if getattr(self, "owned", False) and self.h:
            self.lib.L.ref_hier_free(self.h)

    @property
    def num_levels(self) -> int:
        return self.lib.L.ref_hier_num_levels(self.h)

    def level(self, lev: int) -> Level:
        n, nnz, nc = _i(), C.c_longlong(), _i()
        self.lib.L.ref_hier_level_sizes(self.h, lev, C.byref(n), C.byref(nnz), C.byref(nc))
        rp = np.empty(n.value + 1, np.int32)
        ci = np.empty(nnz.value, np.int32)
        vv = np.empty(nnz.value, np.float64)
        last = lev + 1 == self.num_levels
        agg = None if last else np.empty(n.value, np.int32)
        self.lib.L.ref_hier_level_copy(self.h, lev, rp, ci, vv, None if agg is None else agg.ctypes.data_as(_vp))
        return Level(Csr(n.value, n.value, rp, ci, vv), agg, nc.value)

    def levels(self):
        return [self.level(i) for i in range(self.num_levels)]

    def coarse_lu(self):
        n, nl, nu = _i(), C.c_longlong(), C.c_longlong()
        self.lib.L.ref_hier_coarse_lu_sizes(self.h, C.byref(n), C.byref(nl), C.byref(nu))
        n = n.value
        lrp, lci, lv = np.empty(n + 1, np.int32), np.empty(nl.value, np.int32), np.empty(nl.value)
        urp, uci, uv = np.empty(n + 1, np.int32), np.empty(nu.value, np.int32), np.empty(nu.value)
        perm = np.empty(n, np.int32)
        self.lib.L.ref_hier_coarse_lu_copy(self.h, lrp, lci, lv, urp, uci, uv, perm)
        return Csr(n, n, lrp, lci, lv), Csr(n, n, urp, uci, uv), perm

    def vcycle(self, r):
        r = _f64(r)
        z = np.empty_like(r)
        self.lib._check(self.lib.L.ref_hier_vcycle(self.h, r, z))
        return z


class RefTd:
    """td_bj / td_bgs(Uzawa(AMG_V), AMG_D') wired as bench.cpp:121-182."""

    def __init__(self, lib: RefLib, s: System, kind, v_max_levels, d_max_levels):
        self.lib = lib
        self.sys = s
        self.h = _vp()
        k = {"td_bj": 0, "td_bgs": 1, "td_bj_ilu0": 2, "td_bgs_ilu0": 3}[kind]
        t0 = time.perf_counter()
        lib._check(lib.L.ref_td_new(s.n, s.a.rowptr, s.a.col, s.a.val, s.n_u, s.n_vel, s.n_pff, s.n_ppm,
                                    k, v_max_levels, d_max_levels, C.byref(self.h)))
        self.wall_setup = time.perf_counter() - t0

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.L.ref_td_free(self.h)

    @property
    def omega(self) -> float:
        return self.lib.L.ref_td_omega(self.h)

    @property
    def setup_seconds(self) -> float:
        return self.lib.L.ref_td_setup_seconds(self.h)

    @property
    def v_hierarchy(self) -> RefHierarchy:
        return RefHierarchy(self.lib, self.lib.L.ref_td_v_hier(self.h), owned=False, parent=self)

    @property
    def d_hierarchy(self) -> RefHierarchy:
        return RefHierarchy(self.lib, self.lib.L.ref_td_d_hier(self.h), owned=False, parent=self)

    def apply(self, r):
        r = _f64(r)
        z = np.empty_like(r)
        self.lib._check(self.lib.L.ref_td_apply(self.h, r, z))
        return z

    def uzawa_apply(self, r_ff):
        r = _f64(r_ff)
        z = np.empty_like(r)
        self.lib._check(self.lib.L.ref_uzawa_apply(self.h, r, z))
        return z


# ---------------------------------------------------------------------------
# plain-C restatement (oracle/sdc_oracle.c)


class _OCsr(C.Structure):
    _fields_ = [("n_rows", _i), ("n_cols", _i), ("rp", C.POINTER(_i)), ("ci", C.POINTER(_i)),
                ("v", C.POINTER(_d))]


class _OLevel(C.Structure):
    _fields_ = [("a", _OCsr), ("agg", C.POINTER(_i)), ("n_coarse", _i)]


class _OHier(C.Structure):
    _fields_ = [("n_levels", _i), ("levels", C.POINTER(_OLevel)), ("lower", _OCsr), ("upper", _OCsr),
                ("perm", C.POINTER(_i))]


class _ORestart(C.Structure):
    _fields_ = [("m_init", _i), ("m_min", _i), ("m_step", _i), ("m_max", _i), ("current_m", _i),
                ("previous_rate", _d), ("has_rate_sample", _i), ("alpha_p", _d), ("alpha_d", _d),
                ("stall_threshold", _d)]


class _OReport(C.Structure):
    _fields_ = [("iterations", _i), ("converged", _i), ("final_residual", _d), ("history", C.POINTER(_d)),
                ("capacity", _i), ("length", _i)]


class _OTd(C.Structure):
    _fields_ = [("v", C.POINTER(_OHier)), ("c", C.POINTER(_OCsr)), ("omega", _d), ("c_prime", C.POINTER(_OCsr)),
                ("d", C.POINTER(_OHier)), ("n_v", _i), ("n_pff", _i), ("n_ppm", _i)]


class OCsr:
    """Keeps numpy arrays alive behind an orc_csr view."""

    def __init__(self, a: Csr):
        self.rp, self.ci, self.v = _i32(a.rowptr), _i32(a.col), _f64(a.val)
        if self.v.size == 0:
            self.ci, self.v = np.zeros(1, np.int32), np.zeros(1)
        self.s = _OCsr(a.n_rows, a.n_cols, self.rp.ctypes.data_as(C.POINTER(_i)),
                       self.ci.ctypes.data_as(C.POINTER(_i)), self.v.ctypes.data_as(C.POINTER(_d)))


class OHier:
    """orc_hierarchy view of a reference hierarchy (levels + coarse LU)."""

    def __init__(self, levels, lower: Csr, upper: Csr, perm):
        self.keep = []
        arr = (_OLevel * len(levels))()
        for k, lv in enumerate(levels):
            oc = OCsr(lv.a)
            self.keep.append(oc)
            agg = None
            if lv.aggregate_of is not None:
                agg = _i32(lv.aggregate_of)
                self.keep.append(agg)
            arr[k] = _OLevel(oc.s, None if agg is None else agg.ctypes.data_as(C.POINTER(_i)), lv.n_coarse)
        self.lo, self.up, self.perm = OCsr(lower), OCsr(upper), _i32(perm)
        self.arr = arr
        self.s = _OHier(len(levels), arr, self.lo.s, self.up.s, self.perm.ctypes.data_as(C.POINTER(_i)))

    @staticmethod
    def from_ref(h: "RefHierarchy") -> "OHier":
        lo, up, perm = h.coarse_lu()
        return OHier(h.levels(), lo, up, perm)


class PortLib:
    """The plain-C restatement of the hot path (checker, never the product)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle port`")
        L = C.CDLL(path)
        self.L = L
        P = C.POINTER
        fn = C.CFUNCTYPE(None, _vp, P(_d), P(_d))
        self._fn = fn
        _proto(L, "orc_spmv", None, [P(_OCsr), _dp, _dp])
        _proto(L, "orc_spmv_add", None, [P(_OCsr), _dp, _dp, _d])
        _proto(L, "orc_sor_sweep", _i, [P(_OCsr), _dp, _dp, _d])
        _proto(L, "orc_lu_solve", None, [_i, P(_OCsr), P(_OCsr), _ip, _dp, _dp])
        _proto(L, "orc_aggregate", _i, [P(_OCsr), _d, _vp, _ip])
        _proto(L, "orc_vcycle", _i, [P(_OHier), _dp, _dp])
        _proto(L, "orc_td_bgs_apply", _i, [P(_OHier), P(_OCsr), _d, P(_OCsr), P(_OHier), _i, _i, _i, _dp, _dp])
        _proto(L, "orc_pd_gmres", _i, [_i, _vp, _vp, _vp, _vp, _dp, _d, _i, _ORestart, _dp, P(_OReport)])
        _proto(L, "orc_bicgstab", _i, [_i, _vp, _vp, _vp, _vp, _dp, _d, _i, _dp, P(_OReport)])
        _proto(L, "orc_power_iteration", _d, [_i, _vp, _vp, _d, _i, C.c_uint, P(_i), P(_i)])
        _proto(L, "orc_random_vector", None, [_i, C.c_uint, _dp])
        _proto(L, "orc_restart_update", None, [P(_ORestart), _d])
        self.cb_spmv = C.cast(L.orc_cb_spmv, _vp)
        self.cb_td = C.cast(L.orc_cb_td_bgs, _vp)
        self.cb_vcycle = C.cast(L.orc_cb_vcycle, _vp)

    def spmv(self, a: Csr, x):
        o = OCsr(a)
        y = np.empty(a.n_rows)
        self.L.orc_spmv(C.byref(o.s), _f64(x), y)
        return y

    def spmv_add(self, a: Csr, x, y, alpha=1.0):
        o = OCsr(a)
        y = _f64(y).copy()
        self.L.orc_spmv_add(C.byref(o.s), _f64(x), y, alpha)
        return y

    def sor_sweep(self, a: Csr, z, r, omega=1.0):
        o = OCsr(a)
        z = _f64(z).copy()
        bad = self.L.orc_sor_sweep(C.byref(o.s), z, _f64(r), omega)
        if bad >= 0:
            raise RuntimeError(f"sor_sweep: zero diagonal in row {bad}")
        return z

    def lu_solve(self, lower: Csr, upper: Csr, perm, b):
        lo, up = OCsr(lower), OCsr(upper)
        y = np.empty(lower.n_rows)
        self.L.orc_lu_solve(lower.n_rows, C.byref(lo.s), C.byref(up.s), _i32(perm), _f64(b), y)
        return y

    def aggregate(self, a: Csr, theta=0.08, components=None):
        o = OCsr(a)
        agg = np.empty(a.n_rows, np.int32)
        comp = None if components is None else _i32(components)
        n = self.L.orc_aggregate(C.byref(o.s), theta, None if comp is None else comp.ctypes.data_as(_vp), agg)
        return agg, n

    def vcycle(self, h: OHier, r):
        r = _f64(r)
        z = np.empty_like(r)
        err = self.L.orc_vcycle(C.byref(h.s), r, z)
        if err:
            raise RuntimeError(f"sor_sweep: zero diagonal in row {err - 1}")
        return z

    def td_bundle(self, v: OHier, c: Csr, omega: float, c_prime: Csr, d: OHier, n_v, n_pff, n_ppm):
        oc, ocp = OCsr(c), OCsr(c_prime)
        b = _OTd(C.pointer(v.s), C.pointer(oc.s), omega, C.pointer(ocp.s), C.pointer(d.s), n_v, n_pff, n_ppm)
        b._keep = (v, d, oc, ocp)
        return b

    def td_bgs_apply(self, bundle: "_OTd", r):
        r = _f64(r)
        z = np.empty_like(r)
        err = self.L.orc_td_bgs_apply(bundle.v, bundle.c, bundle.omega, bundle.c_prime, bundle.d, bundle.n_v,
                                      bundle.n_pff, bundle.n_ppm, r, z)
        if err:
            raise RuntimeError("sor_sweep: zero diagonal")
        return z

    def _pre(self, pre):
        if pre is None:
            return None, None
        if isinstance(pre, _OTd):
            return self.cb_td, C.cast(C.pointer(pre), _vp)
        if isinstance(pre, OHier):
            return self.cb_vcycle, C.cast(C.pointer(pre.s), _vp)
        raise TypeError(pre)

    def pd_gmres(self, a: Csr, b, tol_abs, max_restarts, precond=None, m_init=3, m_min=3, m_step=5, m_max=53,
                 hist_cap=1 << 16):
        o = OCsr(a)
        pf, pu = self._pre(precond)
        x = np.empty(a.n_rows)
        hist = np.empty(hist_cap)
        rep = _OReport(0, 0, 0.0, hist.ctypes.data_as(C.POINTER(_d)), hist_cap, 0)
        ctrl = _ORestart(m_init, m_min, m_step, m_max, m_init, 0.0, 0, -3.0, 5.0, 0.05)
        st = self.L.orc_pd_gmres(a.n_rows, self.cb_spmv, C.cast(C.pointer(o.s), _vp), pf, pu, _f64(b), tol_abs,
                                 max_restarts, ctrl, x, C.byref(rep))
        if st:
            raise RuntimeError("pd_gmres: singular Hessenberg block")
        return x, SolveReport(rep.iterations, rep.final_residual, bool(rep.converged), 0.0,
                              hist[: min(rep.length, hist_cap)].copy())

    def bicgstab(self, a: Csr, b, tol_abs, max_iters, precond=None, hist_cap=1 << 16):
        o = OCsr(a)
        pf, pu = self._pre(precond)
        x = np.empty(a.n_rows)
        hist = np.empty(hist_cap)
        rep = _OReport(0, 0, 0.0, hist.ctypes.data_as(C.POINTER(_d)), hist_cap, 0)
        st = self.L.orc_bicgstab(a.n_rows, self.cb_spmv, C.cast(C.pointer(o.s), _vp), pf, pu, _f64(b), tol_abs,
                                 max_iters, x, C.byref(rep))
        if st:
            raise RuntimeError("bicgstab: repeated breakdown")
        return x, SolveReport(rep.iterations, rep.final_residual, bool(rep.converged), 0.0,
                              hist[: min(rep.length, hist_cap)].copy())

    def power_iteration(self, a: Csr, tol_rel, max_iters, seed):
        o = OCsr(a)
        it, cv = _i(), _i()
        v = self.L.orc_power_iteration(a.n_rows, self.cb_spmv, C.cast(C.pointer(o.s), _vp), tol_rel, max_iters,
                                       seed, C.byref(it), C.byref(cv))
        return v, it.value, bool(cv.value)

    def random_vector(self, n, seed):
        out = np.empty(n)
        self.L.orc_random_vector(n, seed, out)
        return out
