"""Strip-sharded multi-GPU solve -- Python mirror of the
`sdg_dist_*` C-ABI.

One process per GPU.  Every rank assembles (or receives) the same global
system, partitions it with :func:`strip_partition` (rank r owns free-flow
strip r from the bottom and porous strip r from the top, so rank 0 holds the
interface), and works on its own rows in ascending global order.  The
library does all device work; communication goes through a transport:

* :class:`NcclTransport` -- the library's built-in NCCL transport (grouped
  ncclSend/ncclRecv halos, ncclAllGather reductions).  The unique id is
  distributed with torch.distributed (the plumbing, not the data path).
* :class:`CallbackTransport` -- host callbacks into torch.distributed (any
  backend that moves CPU tensors, e.g. gloo).  This is what the tests use to
  run two ranks on one GPU, where NCCL refuses a duplicate device.

There is no CPU fallback: every compute call goes through libsdgpu.so.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import sdc
from .sdc import (GmresResult, RestartController, SdgCudaError, SolveReport, _check, _dp, _f64, _i, _i32, _ip,
                  _Report, _Restart, _d, _vp, _report, lib)

_EXCHANGE = C.CFUNCTYPE(_i, _vp, C.POINTER(_d), C.POINTER(_i), C.POINTER(_d), C.POINTER(_i))
_ALLGATHER = C.CFUNCTYPE(_i, _vp, C.POINTER(_d), _i, C.POINTER(_d))

_bound = False


def _lib():
    global _bound
    L = lib()
    if _bound:
        return L

    def p(name, res, args):
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args

    P = C.POINTER
    p("sdg_transport_create_host", _i, [_i, _i, _EXCHANGE, _ALLGATHER, _vp, P(_vp)])
    p("sdg_nccl_get_unique_id", _i, [C.c_char_p])
    p("sdg_transport_create_nccl", _i, [_vp, C.c_char_p, _i, _i, P(_vp)])
    p("sdg_transport_destroy", _i, [_vp])
    p("sdg_strip_partition", _i, [_i, _i, _ip])
    p("sdg_dist_halo_plan", _i, [_i, _ip, _ip, _ip, _i, _i, P(_i), _vp, _vp, P(_i), _vp, _vp])
    p("sdg_dist_system_create", _i, [_vp, _vp, _i, _ip, _ip, _dp, _i, _i, _i, _i, _ip, P(_vp)])
    p("sdg_dist_system_destroy", _i, [_vp])
    p("sdg_dist_local_rows", _i, [_vp, P(_i), _vp])
    p("sdg_dist_spmv", _i, [_vp, _dp, _dp])
    p("sdg_dist_td_create", _i, [_vp, _i, _i, _i, _d, P(_vp)])
    p("sdg_dist_precond_destroy", _i, [_vp])
    p("sdg_dist_precond_omega", _d, [_vp])
    p("sdg_dist_precond_setup_seconds", _d, [_vp])
    p("sdg_dist_precond_apply", _i, [_vp, _vp, _dp, _dp])
    p("sdg_dist_pd_gmres", _i, [_vp, _vp, _dp, _dp, _d, _i, P(_Restart), P(_Report)])
    p("sdg_dist_bicgstab", _i, [_vp, _vp, _dp, _dp, _d, _i, P(_Report)])
    p("sdg_dist_pd_gmres_device", _i, [_vp, _vp, _vp, _vp, _d, _i, P(_Restart), P(_Report)])
    p("sdg_dist_bicgstab_device", _i, [_vp, _vp, _vp, _vp, _d, _i, P(_Report)])
    p("sdg_dist_pd_gmres_warm_device", _i, [_vp, _vp, _vp, _vp, _d, _i, P(_Restart), P(_Report)])
    p("sdg_dist_bicgstab_warm_device", _i, [_vp, _vp, _vp, _vp, _d, _i, P(_Report)])
    _bound = True
    return L


def strip_partition(n: int, size: int) -> np.ndarray:
    """Owner rank of every dof of the n x n monolithic layout (horizontal strips)."""
    nt = 2 * n * (n + 1) + 2 * n * n
    owner = np.empty(nt, dtype=np.int32)
    _check(_lib().sdg_strip_partition(n, size, owner))
    return owner


def halo_plan(a: sdc.SparseMatrix, owner, rank: int, size: int) -> dict:
    """Host-only: the monolithic operator's halo plan on `rank` (no GPU)."""
    L = _lib()
    owner = _i32(owner)
    ng, ns = _i(), _i()
    _check(L.sdg_dist_halo_plan(a.n_rows, a.row_offsets, a.col_indices, owner, rank, size, C.byref(ng), None,
                                None, C.byref(ns), None, None))
    ghost = np.empty(max(ng.value, 1), dtype=np.int32)
    send = np.empty(max(ns.value, 1), dtype=np.int32)
    rc = np.empty(size, dtype=np.int32)
    sc = np.empty(size, dtype=np.int32)
    _check(L.sdg_dist_halo_plan(a.n_rows, a.row_offsets, a.col_indices, owner, rank, size, C.byref(ng),
                                ghost.ctypes.data, rc.ctypes.data, C.byref(ns), send.ctypes.data, sc.ctypes.data))
    return {"ghost_gid": ghost[:ng.value].copy(), "recv_counts": rc, "send_gid": send[:ns.value].copy(),
            "send_counts": sc}


class Transport:
    rank = 0
    size = 1
    h = None

    def __del__(self):
        h = getattr(self, "h", None)
        if h and sdc._lib is not None:
            sdc._lib.sdg_transport_destroy(h)
            self.h = None


class CallbackTransport(Transport):
    """Exchanges through torch.distributed on CPU tensors (e.g. gloo)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self._torch, self._dist, self._group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self._ex = _EXCHANGE(self._exchange)
        self._ag = _ALLGATHER(self._allgather)
        self.h = _vp()
        _check(_lib().sdg_transport_create_host(self.rank, self.size, self._ex, self._ag, None, C.byref(self.h)))

    def _peer(self, p):
        return p if self._group is None else self._dist.get_global_rank(self._group, p)

    def _exchange(self, _user, send, scount, recv, rcount):
        try:
            torch, dist = self._torch, self._dist
            sc = [scount[p] for p in range(self.size)]
            rc = [rcount[p] for p in range(self.size)]
            ns, nr = sum(sc), sum(rc)
            sv = np.ctypeslib.as_array(send, shape=(ns,)) if ns else np.empty(0)
            out = torch.empty(nr, dtype=torch.float64)
            reqs, so, ro = [], 0, 0
            for p in range(self.size):
                if sc[p]:
                    reqs.append(dist.isend(torch.from_numpy(sv[so:so + sc[p]].copy()), self._peer(p), self._group))
                if rc[p]:
                    reqs.append(dist.irecv(out[ro:ro + rc[p]], self._peer(p), self._group))
                so += sc[p]
                ro += rc[p]
            for q in reqs:
                q.wait()
            if nr:
                np.ctypeslib.as_array(recv, shape=(nr,))[:] = out.numpy()
            return 0
        except Exception as e:  # noqa: BLE001 -- reported through the C return code
            print(f"[rank {self.rank}] transport exchange failed: {e!r}")
            return 1

    def _allgather(self, _user, send, count, recv):
        try:
            torch, dist = self._torch, self._dist
            t = torch.from_numpy(np.ctypeslib.as_array(send, shape=(count,)).copy()) if count else torch.empty(0, dtype=torch.float64)
            outs = [torch.empty(count, dtype=torch.float64) for _ in range(self.size)]
            dist.all_gather(outs, t, group=self._group)
            if count:
                np.ctypeslib.as_array(recv, shape=(count * self.size,))[:] = torch.cat(outs).numpy()
            return 0
        except Exception as e:  # noqa: BLE001
            print(f"[rank {self.rank}] transport allgather failed: {e!r}")
            return 1


class NcclTransport(Transport):
    """The library's NCCL transport; the unique id travels over torch.distributed."""

    def __init__(self, ctx: sdc.Context, group=None):
        import torch.distributed as dist
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.size = dist.get_world_size(group) if dist.is_initialized() else 1
        uid = C.create_string_buffer(128)
        if self.rank == 0:
            _check(_lib().sdg_nccl_get_unique_id(uid))
        if self.size > 1:
            obj = [uid.raw]
            dist.broadcast_object_list(obj, src=0 if group is None else dist.get_global_rank(group, 0), group=group)
            uid = C.create_string_buffer(obj[0], 128)
        self.h = _vp()
        _check(_lib().sdg_transport_create_nccl(ctx.h, uid, self.rank, self.size, C.byref(self.h)))


class DistSystem:
    """The coupled system on one rank (sdg_dist_system)."""

    def __init__(self, system: sdc.CoupledSystem, transport: Transport, owner=None,
                 ctx: Optional[sdc.Context] = None):
        self.ctx = ctx or sdc.default_context()
        self.transport = transport
        self.system = system
        a = system.matrix
        self.owner = _i32(owner if owner is not None else strip_partition(system.n, transport.size))
        self.h = _vp()
        _check(_lib().sdg_dist_system_create(self.ctx.h, transport.h, a.n_rows, a.row_offsets, a.col_indices,
                                             a.values, system.n_u, system.n_vel, system.n_pff, system.n_ppm,
                                             self.owner, C.byref(self.h)))
        n = _i()
        _check(_lib().sdg_dist_local_rows(self.h, C.byref(n), None))
        self.rows = np.empty(max(n.value, 1), dtype=np.int32)
        _check(_lib().sdg_dist_local_rows(self.h, C.byref(n), self.rows.ctypes.data))
        self.rows = self.rows[:n.value]

    def n_local(self) -> int:
        return int(self.rows.size)

    def local(self, v) -> np.ndarray:
        """This rank's entries of a global vector."""
        return _f64(np.asarray(v)[self.rows])

    def spmv(self, x_local) -> np.ndarray:
        y = np.empty(self.n_local())
        _check(_lib().sdg_dist_spmv(self.h, _f64(x_local), y))
        return y

    def __del__(self):
        h = getattr(self, "h", None)
        if h and sdc._lib is not None:
            sdc._lib.sdg_dist_system_destroy(h)
            self.h = None


class DistTdPreconditioner:
    """td_bgs / td_bj(Uzawa(AMG_V), AMG_D') over strips (sdg_dist_td_create)."""

    def __init__(self, ds: DistSystem, kind: str = "td_bgs", v_max_levels: int = 3, d_max_levels: int = 3,
                 omega: Optional[float] = None):
        self.ds = ds
        # "uzawa" / "amg": the subdomain preconditioners of the partitioned driver
        # (SDG_DIST_UZAWA on a Stokes system with n_ppm = 0, SDG_DIST_AMG on a single matrix)
        k = {"td_bj": int(sdc.BlockPrecondKind.td_bj), "td_bgs": int(sdc.BlockPrecondKind.td_bgs), "uzawa": 32,
             "amg": 33}[kind]
        self.h = _vp()
        _check(_lib().sdg_dist_td_create(ds.h, k, v_max_levels, d_max_levels,
                                         float("nan") if omega is None else float(omega), C.byref(self.h)))

    def omega(self) -> float:
        return _lib().sdg_dist_precond_omega(self.h)

    def setup_seconds(self) -> float:
        return _lib().sdg_dist_precond_setup_seconds(self.h)

    def apply(self, r_local) -> np.ndarray:
        z = np.empty(self.ds.n_local())
        _check(_lib().sdg_dist_precond_apply(self.ds.h, self.h, _f64(r_local), z))
        return z

    def __del__(self):
        h = getattr(self, "h", None)
        if h and sdc._lib is not None:
            sdc._lib.sdg_dist_precond_destroy(h)
            self.h = None


def dist_pd_gmres(ds: DistSystem, precond: Optional[DistTdPreconditioner], b_local, tol_abs: float,
                  max_restarts: int, ctrl: Optional[RestartController] = None,
                  history_capacity: int = 1 << 16) -> GmresResult:
    """pd_gmres (krylov.cpp:47-184) over strips; collective over the ranks."""
    b = _f64(b_local)
    if b.size != ds.n_local():
        raise ValueError("pd_gmres: dimension mismatch")
    ctrl = ctrl or RestartController.defaults()
    x = np.empty(ds.n_local())
    hist = np.empty(history_capacity)
    rep = _Report()
    rep.residual_history = hist.ctypes.data_as(C.POINTER(_d))
    rep.history_capacity = history_capacity
    rc = ctrl._c()
    _check(_lib().sdg_dist_pd_gmres(ds.h, precond.h if precond else None, b, x, tol_abs, max_restarts,
                                    C.byref(rc), C.byref(rep)))
    return GmresResult(x, _report(rep, hist))


def dist_bicgstab(ds: DistSystem, precond: Optional[DistTdPreconditioner], b_local, tol_abs: float,
                  max_iters: int, history_capacity: int = 1 << 16) -> GmresResult:
    """bicgstab (krylov.cpp:186-292) over strips; collective over the ranks."""
    b = _f64(b_local)
    if b.size != ds.n_local():
        raise ValueError("bicgstab: dimension mismatch")
    x = np.empty(ds.n_local())
    hist = np.empty(history_capacity)
    rep = _Report()
    rep.residual_history = hist.ctypes.data_as(C.POINTER(_d))
    rep.history_capacity = history_capacity
    _check(_lib().sdg_dist_bicgstab(ds.h, precond.h if precond else None, b, x, tol_abs, max_iters, C.byref(rep)))
    return GmresResult(x, _report(rep, hist))


def dist_solve_device(ds: DistSystem, precond: Optional[DistTdPreconditioner], solver: str, b_ptr: int,
                      x_ptr: int, tol_abs: float, max_iters: int,
                      ctrl: Optional[RestartController] = None, warm: bool = False) -> SolveReport:
    """Device-pointer solve over strips (b, x: this rank's rows on its GPU).
    warm: x holds the previous solution; the reference solve of the correction
    (BASELINE config 4 over strips)."""
    rep = _Report()
    hist = np.empty(1 << 14)
    rep.residual_history = hist.ctypes.data_as(C.POINTER(_d))
    rep.history_capacity = hist.size
    ph = precond.h if precond else None
    if solver == "bicgstab":
        f = _lib().sdg_dist_bicgstab_warm_device if warm else _lib().sdg_dist_bicgstab_device
        _check(f(ds.h, ph, b_ptr, x_ptr, tol_abs, max_iters, C.byref(rep)))
    else:
        rc = (ctrl or RestartController.defaults())._c()
        f = _lib().sdg_dist_pd_gmres_warm_device if warm else _lib().sdg_dist_pd_gmres_device
        _check(f(ds.h, ph, b_ptr, x_ptr, tol_abs, max_iters, C.byref(rc), C.byref(rep)))
    return _report(rep, hist)


__all__ = ["dist_solve_device", "dist_bicgstab", "strip_partition", "halo_plan", "CallbackTransport", "NcclTransport", "DistSystem",
           "DistTdPreconditioner", "dist_pd_gmres", "SdgCudaError", "SolveReport"]
