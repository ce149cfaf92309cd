"""Host drivers around the GPU solve (they stay host-side).

:class:`TransientDriver` mirrors ``MonolithicDriver::advance``
(/root/reference/proj/core/src/bench.cpp:183-238) for BASELINE config 4:
implicit Euler, per step ``assemble_monolithic(grid, cfg, v_prev, t)``
(assembly.cpp:327-380) and a preconditioned GMRES solve, ``v_prev`` = the
velocity block of the new solution.  Two documented differences, both
SURVEY.md §8(d):

* the matrix is step-invariant (only the right-hand side sees ``v_prev`` and
  ``t``), so the td_bgs preconditioner is built once instead of per step;
* the stop rule is ``1e-8 * ||b||`` (the reference's ``10 x direct residual``
  needs a banded LU that is infeasible at 1000^2), and with ``warm_start``
  each solve starts from the previous step's solution -- exactly the
  reference solve of the correction (``sdg_pd_gmres_warm`` /
  ``sdg_bicgstab_warm``).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import scenarios, sdc


@dataclass
class StepResult:
    t: float
    iterations: int
    converged: bool
    final_residual: float
    tol: float
    solve_seconds: float
    assembly_seconds: float
    breakdown_restarts: int = 0


@dataclass
class TransientDriver:
    cfg: scenarios.Config
    warm_start: bool = True
    ctrl: Optional[sdc.RestartController] = None
    ctx: Optional[sdc.Context] = None
    x: Optional[np.ndarray] = None
    precond: Optional[sdc.TdPreconditioner] = None
    system: Optional[sdc.CoupledSystem] = None
    history: List[StepResult] = field(default_factory=list)
    max_breakdown_restarts: int = 3
    # checker aid (tests, scripts/ref_spread_c4.py): every step's right-hand side is multiplied
    # element-wise by (1 + 2^-52 u), u ~ U(-1, 1) from this seed -- a rounding-level change of the input
    rhs_perturbation_seed: Optional[int] = None

    def __post_init__(self):
        if not math.isfinite(self.cfg.dt):
            raise ValueError("TransientDriver: the config is stationary (dt = inf)")
        self._rng = None if self.rhs_perturbation_seed is None else np.random.default_rng(self.rhs_perturbation_seed)
        self.ctx = self.ctx or sdc.default_context()
        self.ctrl = self.ctrl or (sdc.RestartController.fixed(50) if self.cfg.solver == "gmres50"
                                  else sdc.RestartController.defaults())

    def advance(self, t: float) -> StepResult:
        import time
        t0 = time.perf_counter()
        v_prev = None if self.x is None else self.x[: self.system.n_vel]
        s = scenarios.build_system(self.cfg, t=t, v_prev=v_prev)
        t_asm = time.perf_counter() - t0
        if self._rng is not None:
            s.rhs = s.rhs * (1.0 + np.ldexp(self._rng.uniform(-1.0, 1.0, s.rhs.size), -52))
        if self.precond is None:
            self.precond = sdc.TdPreconditioner(s, "td_bgs", self.cfg.v_max_levels, self.cfg.d_max_levels,
                                                ctx=self.ctx)
        self.system = s
        tol = 1e-8 * float(np.linalg.norm(s.rhs))
        t1 = time.perf_counter()
        warm = self.warm_start and self.x is not None
        restarts = 0
        if self.cfg.solver == "bicgstab":
            # warm form always (x0 = 0 first): a repeated breakdown -- the shadow
            # residual turning exactly orthogonal to r, which the reference answers
            # by throwing (krylov.cpp:215) -- restarts from the last iterate
            x0 = self.x if warm else np.zeros(s.n_total())
            res = sdc.bicgstab_warm(s.matrix, self.precond, s.rhs, x0, tol, 20000)
            its = res.report.iterations
            while res.report.breakdown and restarts < self.max_breakdown_restarts:
                restarts += 1
                res = sdc.bicgstab_warm(s.matrix, self.precond, s.rhs, res.x, tol, 20000)
                its += res.report.iterations
            res.report.iterations = its
        else:
            res = (sdc.pd_gmres_warm(s.matrix, self.precond, s.rhs, self.x, tol, 4000, self.ctrl) if warm
                   else sdc.pd_gmres(s.matrix, self.precond, s.rhs, tol, 4000, self.ctrl))
        self.x = res.x
        out = StepResult(t, res.report.iterations, res.report.converged, res.report.final_residual, tol,
                         time.perf_counter() - t1, t_asm, restarts)
        self.history.append(out)
        return out

    def run(self, steps: Optional[int] = None) -> List[StepResult]:
        for k in range(1, (steps or self.cfg.steps) + 1):
            self.advance(k * self.cfg.dt)
        return self.history


@dataclass
class CouplingResult:
    converged: bool
    coupling_iterations: int
    inner_iterations: int
    measure_p: List[float]
    measure_v: List[float]
    stokes_iterations: List[int]
    darcy_iterations: List[int]
    solution: Optional[np.ndarray]
    seconds: float
    solve_seconds: float


@dataclass
class PartitionedDriver:
    """CouplingDriver::coupled_timestep (coupling.cpp:252-332) for BASELINE
    config 5: Dirichlet-Neumann alternation of the free-flow problem
    (assemble_stokes with Dirichlet interface velocities, solved by PD-GMRES +
    inexact Uzawa(AMG_V), coupling.cpp:115-138,199-203,218-229) and the porous
    problem (assemble_darcy with Dirichlet interface pressures, BiCGSTAB +
    AMG, coupling.cpp:140-146,204-206,231-242), with the reference's interface
    update: relaxation 0.5 on the first iteration, then IQN-ILS
    (coupling.cpp:45-101, :309-314) -- or, with ``acceleration="relaxation"``,
    the constant under-relaxation ``v += relaxation * R`` every iteration.
    Convergence: both relative interface measures below epsilon
    (coupling.cpp:284-296).  The two matrices do not depend on the interface
    data (only the right-hand sides do), so both preconditioners are built
    once, as the reference's caches do.  Inner stop rule ``inner_tol_rel *
    ||b||`` (the reference's ``10 x direct residual`` needs banded LUs,
    SURVEY.md §8(d))."""

    cfg: sdc.ScenarioConfig
    levels: int = 3
    acceleration: str = "iqn_ils"
    relaxation: float = 0.5
    epsilon: float = 1e-8
    zero_guard: float = 1e-14
    max_coupling_iterations: int = 100
    history_capacity: int = 50
    filter_tolerance: float = 1e-13
    inner_tol_rel: float = 1e-10
    ctx: Optional[sdc.Context] = None
    log: Optional[object] = None  # callable(k, stokes_its, darcy_its, dp_rel, dv_rel, seconds)

    def __post_init__(self):
        self.ctx = self.ctx or sdc.default_context()
        n = self.cfg.cells_per_unit_square
        self.n = n
        self.mu = self.cfg.kinematic_viscosity * self.cfg.density
        z = np.zeros(n)
        # the interface data enter only the right-hand sides: assemble once,
        # then write v_gamma into the Dirichlet rows (assembly.cpp:137-141) and
        # 2 (K/mu) p_gamma into the top Darcy rows (:268-270) per iteration --
        # exactly the values a re-assembly produces (tests/test_gpu_partitioned.py)
        self.stokes_matrix, self.stokes_rhs0 = sdc.assemble_stokes(self.cfg, z)
        self.darcy_matrix, _ = sdc.assemble_darcy(self.cfg, z)
        self.t2 = 2.0 * (self.cfg.permeability / self.mu)
        n_u = n * (n + 1)
        n_vel = 2 * n_u
        nt = self.stokes_matrix.n_rows
        a = self.stokes_matrix
        comps = [0] * n_u + [1] * n_u
        ucfg = sdc.UzawaConfig(amg=sdc.AmgOptions(max_levels=self.levels, components=comps))
        self.stokes_pre = sdc.UzawaPreconditioner(sdc.submatrix(a, 0, n_vel, 0, n_vel),
                                                  sdc.submatrix(a, 0, n_vel, n_vel, nt),
                                                  sdc.submatrix(a, n_vel, nt, 0, n_vel), ucfg, ctx=self.ctx)
        self.darcy_pre = sdc.AmgPreconditioner(self.darcy_matrix, sdc.AmgOptions(max_levels=self.levels),
                                               ctx=self.ctx)
        self.trace_v = np.zeros(n)
        self.trace_p = np.zeros(n)

    def stokes_rhs(self, v_gamma) -> np.ndarray:
        b = self.stokes_rhs0.copy()
        n_u = self.n * (self.n + 1)
        b[n_u:n_u + self.n] = v_gamma
        return b

    def darcy_rhs(self, p_gamma) -> np.ndarray:
        b = np.zeros(self.darcy_matrix.n_rows)
        b[(self.n - 1) * self.n:] = self.t2 * np.asarray(p_gamma, dtype=np.float64)
        return b

    def solve_ff(self, v_gamma):
        b = self.stokes_rhs(v_gamma)
        res = sdc.pd_gmres(self.stokes_matrix, self.stokes_pre, b, self.inner_tol_rel * float(np.linalg.norm(b)),
                           400, sdc.RestartController.defaults())
        if not res.report.converged:
            raise RuntimeError(f"coupling: inner free-flow solve did not converge, final residual "
                               f"{res.report.final_residual} after {res.report.iterations} iterations")
        return res, sdc.stokes_pressure_trace(self.cfg, res.x)

    def solve_pm(self, p_gamma):
        b = self.darcy_rhs(p_gamma)
        res = sdc.bicgstab(self.darcy_matrix, self.darcy_pre, b, self.inner_tol_rel * float(np.linalg.norm(b)),
                           10000)
        if not res.report.converged:
            raise RuntimeError(f"coupling: inner porous solve did not converge, final residual "
                               f"{res.report.final_residual} after {res.report.iterations} iterations")
        return res, sdc.darcy_velocity_trace(self.cfg, res.x, p_gamma)

    def coupled_step(self) -> CouplingResult:
        import time
        from .iqn import IqnIlsHistory, iqn_ils_update
        t0 = time.perf_counter()
        solve_s = 0.0
        v_k, p_k = self.trace_v.copy(), self.trace_p.copy()
        hist = IqnIlsHistory(self.history_capacity, self.filter_tolerance)
        out = CouplingResult(False, 0, 0, [], [], [], [], None, 0.0, 0.0)

        def measure(nxt, prev):
            return float(np.linalg.norm(nxt - prev)), float(np.linalg.norm(nxt))

        for k in range(self.max_coupling_iterations):
            s0 = time.perf_counter()
            ff, p_tr = self.solve_ff(v_k)
            pm, v_tr = self.solve_pm(p_tr)
            solve_s += time.perf_counter() - s0
            out.coupling_iterations += 1
            out.stokes_iterations.append(ff.report.iterations)
            out.darcy_iterations.append(pm.report.iterations)
            out.inner_iterations += ff.report.iterations + pm.report.iterations
            dp, np_ = measure(p_tr, p_k)
            dv, nv = measure(v_tr, v_k)
            out.measure_p.append(dp)
            out.measure_v.append(dv)
            if self.log:
                self.log(k, ff.report.iterations, pm.report.iterations, dp / max(np_, 1e-300), dv / max(nv, 1e-300),
                         time.perf_counter() - t0)
            zg = self.zero_guard
            ok_p = dp < zg if np_ < zg else dp < self.epsilon * np_
            ok_v = dv < zg if nv < zg else dv < self.epsilon * nv
            if ok_p and ok_v or k + 1 == self.max_coupling_iterations:
                out.converged = bool(ok_p and ok_v)
                out.solution = np.concatenate([ff.x, pm.x])
                if out.converged:
                    self.trace_v, self.trace_p = v_tr, p_tr
                break
            residual = v_tr - v_k
            if self.acceleration == "picard":
                v_next = v_tr
            elif self.acceleration == "relaxation":
                v_next = v_k + self.relaxation * residual
            elif not hist.has_previous():
                v_next = v_k + self.relaxation * residual
                hist.record(residual, v_tr)
            else:
                v_next = iqn_ils_update(hist, v_k, residual, v_tr)
            p_k, v_k = p_tr, v_next
        out.seconds = time.perf_counter() - t0
        out.solve_seconds = solve_s
        return out


@dataclass
class ShardedPartitionedDriver(PartitionedDriver):
    """BASELINE config 5 with the two subdomain solves sharded over horizontal
    strips (one rank per GPU): PD-GMRES + inexact Uzawa(AMG_V) on the Stokes
    box and BiCGSTAB + AMG on the Darcy box through the ``sdg_dist_*`` entry
    points (``SDG_DIST_UZAWA`` / ``SDG_DIST_AMG``).  The coupling loop, the
    traces and IQN-ILS stay on the host and are replicated: rank 0 owns both
    strips at the interface (``strip_partition``), so it evaluates the traces
    (assembly.cpp:382-402 read only cells next to the interface) and
    broadcasts them; every rank then takes the same decisions.  The interface
    data change only right-hand-side rows that rank 0 owns.

    ``transport``: a :class:`paper_2108_13229_b200.dist.Transport`.
    ``solution`` of the result is this rank's rows of [x_ff | p_pm]
    (``local_rows()`` gives their global ids)."""

    transport: Optional[object] = None

    def __post_init__(self):
        from . import dist as sd
        import torch.distributed as td
        if self.transport is None:
            raise ValueError("ShardedPartitionedDriver: a transport is required")
        self._td = td
        self.ctx = self.ctx or sdc.default_context()
        n = self.cfg.cells_per_unit_square
        self.n = n
        self.mu = self.cfg.kinematic_viscosity * self.cfg.density
        z = np.zeros(n)
        self.stokes_matrix, self.stokes_rhs0 = sdc.assemble_stokes(self.cfg, z)
        self.darcy_matrix, _ = sdc.assemble_darcy(self.cfg, z)
        self.t2 = 2.0 * (self.cfg.permeability / self.mu)
        n_u = n * (n + 1)
        n_vel, n_p = 2 * n_u, n * n
        owner = sd.strip_partition(n, self.transport.size)
        if self.transport.size > 1 and n // self.transport.size < 2:
            raise ValueError("ShardedPartitionedDriver: strips need at least two cell rows")
        ff = sdc.CoupledSystem(self.stokes_matrix, self.stokes_rhs0, n, n_u, n_vel, n_p, 0)
        pm = sdc.CoupledSystem(self.darcy_matrix, np.zeros(n_p), n, 0, 0, 0, n_p)
        self.ds_ff = sd.DistSystem(ff, self.transport, owner=owner[: n_vel + n_p], ctx=self.ctx)
        self.ds_pm = sd.DistSystem(pm, self.transport, owner=owner[n_vel + n_p:], ctx=self.ctx)
        self.stokes_pre = sd.DistTdPreconditioner(self.ds_ff, "uzawa", v_max_levels=self.levels)
        self.darcy_pre = sd.DistTdPreconditioner(self.ds_pm, "amg", d_max_levels=self.levels)
        self.trace_v = np.zeros(n)
        self.trace_p = np.zeros(n)

    def local_rows(self):
        """Global ids (in [x_ff | p_pm]) of this rank's entries of ``solution``."""
        return np.concatenate([self.ds_ff.rows, self.stokes_matrix.n_rows + self.ds_pm.rows])

    def _norm(self, v_local) -> float:
        """Global 2-norm of a distributed vector (partials folded in rank order on every rank)."""
        import torch
        part = torch.tensor([float(np.dot(v_local, v_local))], dtype=torch.float64)
        parts = [torch.zeros(1, dtype=torch.float64) for _ in range(self.transport.size)]
        self._gather(parts, part)
        return float(np.sqrt(sum(float(p[0]) for p in parts)))

    def _gather(self, outs, t):
        td = self._td
        if td.get_backend() == "nccl":
            import torch
            dev = torch.device("cuda", torch.cuda.current_device())
            o = [x.to(dev) for x in outs]
            td.all_gather(o, t.to(dev))
            for a, b in zip(outs, o):
                a.copy_(b.cpu())
        else:
            td.all_gather(outs, t)

    def _bcast0(self, arr) -> np.ndarray:
        """Rank 0's array on every rank."""
        import torch
        td = self._td
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64).copy())
        if td.get_backend() == "nccl":
            dev = torch.device("cuda", torch.cuda.current_device())
            g = t.to(dev)
            td.broadcast(g, src=0)
            return g.cpu().numpy()
        td.broadcast(t, src=0)
        return t.numpy()

    def _scatter_full(self, ds, x_local, n_total) -> np.ndarray:
        full = np.zeros(n_total)
        full[ds.rows] = x_local
        return full

    def solve_ff(self, v_gamma):
        from . import dist as sd
        b = self.ds_ff.local(self.stokes_rhs(v_gamma))
        res = sd.dist_pd_gmres(self.ds_ff, self.stokes_pre, b, self.inner_tol_rel * self._norm(b), 400,
                               sdc.RestartController.defaults())
        if not res.report.converged:
            raise RuntimeError(f"coupling: inner free-flow solve did not converge, final residual "
                               f"{res.report.final_residual} after {res.report.iterations} iterations")
        # the trace reads p_ff(i, 0), v(i, 0), v(i, 1): rank 0's strip
        tr = sdc.stokes_pressure_trace(self.cfg, self._scatter_full(self.ds_ff, res.x, self.stokes_matrix.n_rows))
        return res, self._bcast0(tr)

    def solve_pm(self, p_gamma):
        from . import dist as sd
        b = self.ds_pm.local(self.darcy_rhs(p_gamma))
        res = sd.dist_bicgstab(self.ds_pm, self.darcy_pre, b, self.inner_tol_rel * self._norm(b), 10000)
        if not res.report.converged:
            raise RuntimeError(f"coupling: inner porous solve did not converge, final residual "
                               f"{res.report.final_residual} after {res.report.iterations} iterations")
        tr = sdc.darcy_velocity_trace(self.cfg, self._scatter_full(self.ds_pm, res.x, self.darcy_matrix.n_rows),
                                      p_gamma)
        return res, self._bcast0(tr)
