#!/usr/bin/env python
"""Benchmark of the B200 preconditioned Krylov path (one JSON line on rank 0).

Metric (BASELINE.json): solve time to 1e-8 rel. residual; DoF*iter/s; SpMV
GB/s vs B200 HBM peak.  `value` is DoF*iterations per second of whole solves
with the right-hand side already resident in HBM; at N > 1 ranks the one
system is split into horizontal strips over the GPUs (strong scaling, SURVEY.md
§8(e); --replicas runs one independent copy per GPU instead); `e2e` is the same metric through the
public host-pointer C-ABI call (sdg_bicgstab / sdg_pd_gmres: host->device copy
of b and device->host copy of x inside the timed region).  One step = one full
preconditioned solve of the workload's system.

Workload (N=1): BASELINE.json configs[2] = "c3": 500 x 500 cells per
subdomain (1,001,000 DoF), K = 1e-2, GMRES(50) with td_bgs(Uzawa(AMG_V),
AMG_D'), 3 AMG levels -- the largest configuration that runs on one GPU and is
pinned against the reference at full size (165 = 165 iterations,
tests/test_gpu_solvers.py).  c4 (one bench step = ten implicit-Euler solves,
minutes) and c5 (partitioned, 16 M DoF) run with --config; c1/c2 are parity
cases.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--gpus N` without RANK/WORLD_SIZE in the environment re-launches itself
through torch.distributed.run with N ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "solve time to 1e-8 rel. residual; DoF·iter/s; SpMV GB/s vs B200 HBM peak"
UNIT = "DoF*iter/s"
FLUSH_BYTES = 256 << 20  # > 126 MB L2


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c3")
    ap.add_argument("--ref-threads", type=int, default=64,
                    help="reference arm: concurrent reference samples (capped at the usable host cores)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--coupling-iterations", type=int, default=0,
                    help="config 5: cap the Dirichlet-Neumann loop (0 = run to convergence)")
    ap.add_argument("--sharded", action="store_true",
                    help="strip-shard one system across the ranks (strong scaling, sdg_dist_*); the default "
                         "for N > 1 ranks")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1 ranks: one independent replica of the workload per GPU (weak scaling) instead "
                         "of the strip-sharded solve")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def job_totals(dist, elapsed, work, device="cpu"):
    """Whole-job totals over ranks (one replica per rank, weak scaling): the
    slowest rank's elapsed time and the summed work.  `dist` is
    torch.distributed (None for a single process); works with NCCL (device
    tensors) and gloo (CPU tensors, the CPU tests)."""
    if dist is None:
        return float(elapsed), float(work)
    import torch
    t = torch.tensor([float(elapsed)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    w = torch.tensor([float(work)], dtype=torch.float64, device=device)
    dist.all_reduce(w, op=dist.ReduceOp.SUM)
    return float(t.item()), float(w.item())


def measured_peak_gbs():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def workload_desc(cfg, n_dof):
    solver = {"bicgstab": "BiCGSTAB", "gmres50": "GMRES(50)", "pdgmres": "PD-GMRES"}[cfg.solver]
    k = "log-normal K (log10 K ~ N(0,1), seed 13229)" if cfg.lognormal else f"K={cfg.permeability:g}"
    return (f"{cfg.name}: {cfg.n}x{cfg.n} cells per subdomain, {n_dof:,} DoF, {k}, {solver} + "
            f"td_bgs(Uzawa(AMG_V), AMG_D'), AMG levels V{cfg.v_max_levels}/D{cfg.d_max_levels}, tol 1e-8*||b||")


def config_for(cfg, n_dof, nnz, args):
    """The `config` object of the JSON line: static facts of the workload and
    of the command line only, so both arms (ours and --impl reference) print
    the same object."""
    if args.gpus <= 1 and not args.sharded:
        par = "single GPU"
    elif args.replicas:
        par = f"replicas x{args.gpus}"
    else:
        par = f"horizontal strips x{args.gpus} (processor-block GS inside strips, NCCL halos)"
    return {"workload": workload_desc(cfg, n_dof), "dof": int(n_dof), "nnz": int(nnz), "parallelism": par,
            "l2": "GPU arm: flushed between timed solves (256 MiB write, outside the event pair); the working set "
                  "(operator, hierarchy, coarse inverse, interface response) also exceeds the 126 MB L2"}


def solve_device(sdc, cfg, s, p, b_ptr, x_ptr, tol, ctx):
    if cfg.solver == "bicgstab":
        return sdc.bicgstab_device(s.matrix, p, b_ptr, x_ptr, tol, 20000, ctx=ctx)
    ctrl = sdc.RestartController.fixed(50) if cfg.solver == "gmres50" else sdc.RestartController.defaults()
    return sdc.pd_gmres_device(s.matrix, p, b_ptr, x_ptr, tol, 4000, ctrl, ctx=ctx)


def solve_host(sdc, cfg, s, p, b, tol):
    if cfg.solver == "bicgstab":
        return sdc.bicgstab(s.matrix, p, b, tol, 20000)
    ctrl = sdc.RestartController.fixed(50) if cfg.solver == "gmres50" else sdc.RestartController.defaults()
    return sdc.pd_gmres(s.matrix, p, b, tol, 4000, ctrl)


def host_cpu():
    """CPU model and core counts of this host (for the cpu_baseline records)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        usable = os.cpu_count()
    return {"cpu_model": model, "host_logical_cpus": os.cpu_count(), "usable_cpus": usable}


def ref_system_for(R, cfg):
    """The workload's system on the reference side.  Uniform K, stationary
    (c1, c2u, c3): the reference's own assemble_monolithic (oracle harness
    ref_system_new) -- no repo code is loaded.  The log-normal field (c2, c4)
    is an extension the reference cannot express: the repo's host assembly,
    bitwise the reference's for uniform K (tests/test_host.py), builds it."""
    from oracle.refpy import Csr, System
    if not cfg.lognormal and math.isinf(cfg.dt):
        return R.assemble(cfg.n, permeability=cfg.permeability), "reference assemble_monolithic (oracle/_ref)"
    from paper_2108_13229_b200 import scenarios
    s = scenarios.build_system(cfg)
    n = s.n_total()
    return (System(n, s.n_u, s.n_vel, s.n_pff, s.n_ppm,
                   Csr(n, n, s.matrix.row_offsets, s.matrix.col_indices, s.matrix.values), s.rhs),
            "repo host assembly (log-normal K extension; bitwise the reference for uniform K)")


def ref_sample(R, rm, rtd, cfg, b, tol):
    """One bounded step of the reference CPU path on the workload: for
    GMRES(50) its first restart cycle (krylov.cpp:80-167 with max_restarts = 1:
    50 Arnoldi steps, the cycle-end update and the true residual); for
    BiCGSTAB / PD-GMRES the whole solve."""
    if cfg.solver == "bicgstab":
        return R.bicgstab(rm, b, tol, 20000, precond=rtd)
    if cfg.solver == "gmres50":
        return R.pd_gmres(rm, b, tol, 1, precond=rtd, m_init=50, m_min=50, m_max=50)
    return R.pd_gmres(rm, b, tol, 4000, precond=rtd)


SAMPLE_DESC = {"gmres50": "the first GMRES(50) restart cycle (50 Arnoldi steps + cycle end)",
               "bicgstab": "one full BiCGSTAB solve", "pdgmres": "one full PD-GMRES solve"}


class RefSetup:
    """The reference's td_bgs setup (amg_setup + coarse lu_factor + power
    iteration) on its own system, started in a background thread: the ctypes
    call releases the GIL, so it overlaps the GPU measurement (c3's coarse
    lu_factor alone takes minutes on one core)."""

    def __init__(self, cfg):
        from oracle.refpy import RefLib
        self.cfg = cfg
        self.R = RefLib()
        self.error = None
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        try:
            t0 = time.perf_counter()
            self.rs, self.assembly = ref_system_for(self.R, self.cfg)
            self.assembly_s = time.perf_counter() - t0
            t0 = time.perf_counter()
            self.rtd = self.R.td(self.rs, "td_bgs", self.cfg.v_max_levels, self.cfg.d_max_levels)
            self.setup_s = time.perf_counter() - t0
        except Exception as e:  # reported in the JSON line
            self.error = f"{type(e).__name__}: {e}"

    def wait(self):
        self.t.join()
        if self.error:
            raise RuntimeError(self.error)
        return self


def cpu_baseline(setup: RefSetup):
    """The reference's own CPU path (oracle/_ref, single-threaded C++) on the
    workload, 1 core: one bounded sample (ref_sample) after its setup."""
    try:
        st = setup.wait()
    except Exception as e:  # pragma: no cover - only when the oracle was not built / failed
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "reference", "sample": f"unavailable: {e}"}
    cfg, R, rs = st.cfg, st.R, st.rs
    from oracle.refpy import RefMatrix
    tol = 1e-8 * float(np.linalg.norm(rs.rhs))
    with RefMatrix(R, rs.a) as rm:
        t0 = time.perf_counter()
        _, rep = ref_sample(R, rm, st.rtd, cfg, rs.rhs, tol)
        secs = time.perf_counter() - t0
    return {"value": rs.n * rep.iterations / secs, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"{SAMPLE_DESC[cfg.solver]} of {cfg.name} by the compiled reference (oracle/_ref, "
                      f"single-threaded), {rep.iterations} iterations; setup {st.setup_s:.1f} s excluded "
                      f"(run in a background thread beside the GPU measurement)",
            "sample_s": secs, "iterations": rep.iterations, "setup_s": st.setup_s, "system": st.assembly,
            **host_cpu()}


def run_reference(args):
    """The reference arm: the unmodified reference CPU path (oracle/_ref,
    compiled from /root/reference by oracle/Makefile) on the same workload,
    on all usable host cores -- independent concurrent samples sharing one
    setup (a Preconditioner is const and reentrant, operator.hpp:30-33), the
    way the reference's own bench runs independent cells on a thread pool
    (bench.cpp:438-457).  Rank 0 only."""
    rank, local_rank, world = dist_env()
    if rank != 0:
        return 0
    from concurrent.futures import ThreadPoolExecutor

    from oracle.refpy import RefMatrix
    from paper_2108_13229_b200 import scenarios
    cfg = scenarios.CONFIGS[args.config]
    st = RefSetup(cfg).wait()
    R, rs = st.R, st.rs
    tol = 1e-8 * float(np.linalg.norm(rs.rhs))
    cpu = host_cpu()
    threads = max(1, min(cpu["usable_cpus"] or 1, args.ref_threads))
    rms = [RefMatrix(R, rs.a) for _ in range(threads)]

    def batch():
        with ThreadPoolExecutor(max_workers=threads) as ex:
            reps = list(ex.map(lambda rm: ref_sample(R, rm, st.rtd, cfg, rs.rhs, tol)[1], rms))
        return sum(r.iterations for r in reps)

    for _ in range(args.warmup):  # untimed; one sample on one core warms the caches as well as a batch
        ref_sample(R, rms[0], st.rtd, cfg, rs.rhs, tol)
    times, its = [], []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        its.append(batch())
        times.append(time.perf_counter() - t0)
    for rm in rms:
        rm.close()
    value = rs.n * sum(its) / sum(times)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": config_for(cfg, rs.n, len(rs.a.val), args),
            "details": {"iterations_per_step": its, "setup_s": st.setup_s, "system": st.assembly},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"each step = {threads} concurrent samples ({SAMPLE_DESC[cfg.solver]} of "
                                       f"{cfg.name}) by the compiled reference, one per core, sharing one setup",
                             **cpu},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def roofline_entry(prof, fam, peak, peak_kind, step_ms, traffic):
    """Achieved algorithmic bytes per launch / mean launch time of one kernel
    family (CUDA events around every launch on its own stream, one profiled
    solve), against the measured HBM peak."""
    f = prof[fam]
    per_launch_ms = f["ms"] / f["launches"]
    per_launch_bytes = f["bytes"] / f["launches"]
    ach = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9
    t = traffic.get(fam)
    return {"kernel": fam, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "peak_source": peak_kind, "traffic": t["dram_bytes_per_launch"] if t else None,
            "traffic_note": (t["kernel"] + "; " + t["source"]) if t else None,
            "bytes_per_launch": per_launch_bytes, "ms_per_launch": per_launch_ms, "launches": f["launches"],
            "share_of_kernel_time": f["ms"] / sum(v["ms"] for v in prof.values()),
            # two streams overlap (td_bgs: the porous V-cycle runs beside the
            # Uzawa one), so family shares of the step can add up to more than 1
            "share_of_step": f["ms"] / step_ms}


def run_ours(args):
    import torch
    rank, local_rank, world = dist_env()
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    torch.cuda.set_device(local_rank)
    from paper_2108_13229_b200 import scenarios, sdc

    cfg = scenarios.CONFIGS[args.config]
    # the reference's own setup for the cpu_baseline, beside the GPU work
    ref_setup = RefSetup(cfg) if (rank == 0 and world == 1 and not args.no_cpu_baseline) else None
    t0 = time.perf_counter()
    s = scenarios.build_system(cfg)
    assembly_s = time.perf_counter() - t0
    n = s.n_total()
    tol = 1e-8 * float(np.linalg.norm(s.rhs))
    ctx = sdc.Context(local_rank)
    t0 = time.perf_counter()
    p = sdc.TdPreconditioner(s, "td_bgs", cfg.v_max_levels, cfg.d_max_levels, ctx=ctx)
    setup_s = time.perf_counter() - t0
    hier_v, hier_d = p.hierarchy(0), p.hierarchy(1)

    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    b_dev = torch.from_numpy(s.rhs).to(dev)
    x_dev = torch.zeros(n, dtype=torch.float64, device=dev)
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    torch.cuda.synchronize()

    def step():
        return solve_device(sdc, cfg, s, p, b_dev.data_ptr(), x_dev.data_ptr(), tol, ctx)

    for _ in range(args.warmup):
        rep = step()
        if not rep.converged:
            raise RuntimeError(f"warm-up solve did not converge: {rep}")

    clocks = ClockSampler(local_rank)
    clocks.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    evs, iters = [], []
    if os.environ.get("SDG_PROFILER_RANGE"):  # ncu --profile-from-start off: the timed solves only
        torch.cuda.profiler.start()
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()  # L2 flush outside the timed pair
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        rep = step()
        with torch.cuda.stream(stream):
            e1.record(stream)
        evs.append((e0, e1))
        iters.append(rep.iterations)
    torch.cuda.synchronize()
    if os.environ.get("SDG_PROFILER_RANGE"):
        torch.cuda.profiler.stop()
    if dist:
        dist.barrier()
    launches = ctx.launches - launches0
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    total_ms, work = job_totals(dist, total_ms, float(n) * sum(iters), dev)
    value = work / (total_ms / 1e3)

    # parity self-check of the timed solve (residual of the returned x)
    x_host = x_dev.cpu().numpy()
    true_res = float(np.linalg.norm(s.rhs - sdc.spmv(s.matrix, x_host)))

    # e2e through the public host-pointer C-ABI call (sdg_pd_gmres / sdg_bicgstab):
    # H2D of b from pinned memory and D2H of x inside the timed region
    e2e = None
    if not args.no_e2e:
        b_pin = torch.from_numpy(s.rhs.copy()).pin_memory()
        b_np = b_pin.numpy()
        solve_host(sdc, cfg, s, p, b_np, tol)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        e_its = 0
        for _ in range(args.steps):
            res = solve_host(sdc, cfg, s, p, b_np, tol)
            e_its += res.report.iterations
        e_s = time.perf_counter() - t0
        e_s, e_work = job_totals(dist, e_s, float(n) * e_its, dev)
        e2e = {"value": e_work / e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
               "ms_per_step": 1e3 * e_s / args.steps, "timing": "host wall clock around the synchronous C-ABI call"}

    # live per-kernel-family profile of one more solve (CUDA events on the
    # stream each kernel is launched on)
    ctx.set_profiling(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
    step()
    with torch.cuda.stream(stream):
        e1.record(stream)
    torch.cuda.synchronize()
    prof_step_ms = e0.elapsed_time(e1)
    prof = ctx.profile()
    ctx.set_profiling(False)
    peak, peak_kind = measured_peak_gbs()
    traffic = {}
    try:  # DRAM bytes per launch from the committed ncu --set full captures (profiles/)
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = {k: v for k, v in json.load(f).items() if v.get("config") == cfg.name}
    except Exception:
        pass
    dominant = max(prof, key=lambda k: prof[k]["ms"])
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_for(cfg, n, s.matrix.nnz(), args),
        "details": {"iterations": iters, "setup_s": setup_s, "assembly_s": assembly_s,
                   "hierarchy_v": hier_v, "hierarchy_d": hier_d, "omega": p.omega(),
                   "fast_paths": sorted(p.features()),
                   "true_residual_rel": true_res / float(np.linalg.norm(s.rhs))},
        "solve_ms": total_ms / args.steps,
        "roofline": roofline_entry(prof, dominant, peak, peak_kind, prof_step_ms, traffic),
        "other_rooflines": {k: roofline_entry(prof, k, peak, peak_kind, prof_step_ms, traffic)
                            for k in ("spmv", "gs_wave", "coarse", "iface", "ortho")
                            if k in prof and k != dominant},
        "kernel_profile": {k: {"launches": v["launches"], "ms": v["ms"], "GBps": v["bytes"] / v["ms"] / 1e6}
                           for k, v in prof.items()},
        "profiled_solve_ms": prof_step_ms,
        "gpu_launches": launches,
        "clocks": clk,
        "e2e": e2e,
    }
    if ref_setup is not None:
        line["cpu_baseline"] = cpu_baseline(ref_setup)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def run_transient(args):
    """BASELINE config 4: implicit Euler x cfg.steps (drivers.TransientDriver
    semantics: rhs re-assembled from the previous velocity -- on the device,
    sdg_assemble_rhs_device --, the preconditioner built once, warm-started
    solves).  One bench step = the
    whole transient run.  `value` = DoF*iterations / device time of the solves
    (CUDA events around each warm-started device solve); `e2e` = the same run
    on the host clock, including host assembly, H2D of each rhs and D2H of each
    solution."""
    import torch
    from paper_2108_13229_b200 import scenarios, sdc
    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    cfg = scenarios.CONFIGS[args.config]
    ctx = sdc.Context(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    t0 = time.perf_counter()
    s1 = scenarios.build_system(cfg, t=cfg.dt)
    assembly_s = time.perf_counter() - t0
    n = s1.n_total()
    t0 = time.perf_counter()
    p = sdc.TdPreconditioner(s1, "td_bgs", cfg.v_max_levels, cfg.d_max_levels, ctx=ctx)
    setup_s = time.perf_counter() - t0
    ctrl = sdc.RestartController.fixed(50)
    b_dev = torch.empty(n, dtype=torch.float64, device=dev)
    x_dev = torch.zeros(n, dtype=torch.float64, device=dev)
    b_pin = torch.empty(n, dtype=torch.float64).pin_memory()
    x_pin = torch.empty(n, dtype=torch.float64).pin_memory()

    def solve(k, tol):
        a, bp, xp = s1.matrix, b_dev.data_ptr(), x_dev.data_ptr()
        if cfg.solver == "bicgstab":
            # warm form throughout (x = 0 before step 1); a repeated breakdown
            # restarts from the last iterate (drivers.TransientDriver)
            rep = sdc.bicgstab_warm_device(a, p, bp, xp, tol, 20000, ctx=ctx)
            its, tries = rep.iterations, 0
            while rep.breakdown and tries < 3:
                tries += 1
                rep = sdc.bicgstab_warm_device(a, p, bp, xp, tol, 20000, ctx=ctx)
                its += rep.iterations
            rep.iterations = its
            return rep
        return (sdc.pd_gmres_device(a, p, bp, xp, tol, 4000, ctrl, ctx=ctx) if k == 0
                else sdc.pd_gmres_warm_device(a, p, bp, xp, tol, 4000, ctrl, ctx=ctx))

    sc = scenarios.scenario(cfg)

    def one_run(log=False):
        ms, its, last_rhs = 0.0, [], None
        x_dev.zero_()
        w0 = time.perf_counter()
        for k in range(cfg.steps):
            # the step's right-hand side from the previous velocity, assembled on
            # the device (sdg_assemble_rhs_device, bitwise the host assembly;
            # the matrix is step-invariant)
            sdc.assemble_rhs_device(sc, b_dev.data_ptr(), None if k == 0 else x_dev.data_ptr(),
                                    t=(k + 1) * cfg.dt, ctx=ctx)
            with torch.cuda.stream(stream):
                bn = float(torch.linalg.vector_norm(b_dev))
            tol = 1e-8 * bn
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
            rep = solve(k, tol)
            with torch.cuda.stream(stream):
                e1.record(stream)
            x_pin.copy_(x_dev)
            torch.cuda.synchronize()
            ms += e0.elapsed_time(e1)
            its.append(rep.iterations)
            if not rep.converged:
                raise RuntimeError(f"time step {k + 1} did not converge: {rep}")
            if log:
                print(f"[c4] step {k + 1}: {rep.iterations} iterations, {e0.elapsed_time(e1):.1f} ms",
                      file=sys.stderr, flush=True)
            last_rhs = b_dev
        return ms, its, time.perf_counter() - w0, last_rhs

    for _ in range(args.warmup):
        one_run()
    clocks = ClockSampler(local_rank)
    clocks.start()
    launches0 = ctx.launches
    total_ms, total_wall, iters = 0.0, 0.0, []
    for _ in range(args.steps):
        ms, its, wall, last_rhs = one_run(log=True)
        total_ms += ms
        total_wall += wall
        iters.append(its)
    launches = ctx.launches - launches0
    clk = clocks.stop()
    work = float(n) * sum(sum(i) for i in iters)
    last_rhs = last_rhs.cpu().numpy()
    true_res = float(np.linalg.norm(last_rhs - sdc.spmv(s1.matrix, x_pin.numpy())))
    line = {
        "metric": METRIC, "value": work / (total_ms / 1e3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_desc(cfg, s1.n_total()) + f", implicit Euler dt={cfg.dt} x{cfg.steps}, warm-started",
                   "dof": n, "nnz": s1.matrix.nnz(), "parallelism": "single GPU",
                   "l2": f"inputs exceed the 126 MB L2 (matrix {12 * s1.matrix.nnz() / 1e6:.0f} MB)",
                   "iterations_per_time_step": iters[-1], "setup_s": setup_s, "assembly_s": assembly_s,
                   "hierarchy_v": p.hierarchy(0), "hierarchy_d": p.hierarchy(1), "omega": p.omega(),
                   "true_residual_rel_last_step": true_res / float(np.linalg.norm(last_rhs))},
        "gpu_launches": launches, "clocks": clk,
        "e2e": {"value": work / total_wall, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 8 * n * cfg.steps, "ms_per_step": 1e3 * total_wall / args.steps,
                "timing": "host wall clock of the run: device assembly of each rhs from the previous velocity, "
                          "device solve, D2H of each solution"},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_partitioned(args):
    """BASELINE config 5: one bench step = one converged Dirichlet-Neumann
    coupling loop (drivers.PartitionedDriver: PD-GMRES + Uzawa(AMG) free-flow
    solves, BiCGSTAB + AMG porous solves, IQN-ILS interface update).  `value`
    = (free-flow DoF x its + porous DoF x its) / time inside the subdomain
    solves (host-pointer C-ABI calls, so this is end to end per solve); `e2e`
    = the same work over the whole loop (host rhs assembly, traces, IQN-ILS)."""
    from paper_2108_13229_b200 import drivers, scenarios, sdc
    rank, local_rank, world = dist_env()
    cfg = scenarios.CONFIGS[args.config]
    sc = scenarios.scenario(cfg)
    sharded = (args.sharded or world > 1) and not args.replicas
    if sharded or world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local_rank)
        if not tdist.is_initialized():
            if world == 1:
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
                os.environ.setdefault("MASTER_PORT", "29533")
            tdist.init_process_group("nccl", rank=rank, world_size=world)
    ctx = sdc.Context(local_rank)
    # inner stop rule relative to ||b||: 1e-12 up to 500^2; at 2000^2 the attainable residual of the
    # 12 M-DoF Stokes solve is ~1e-13 absolute, above 1e-12 ||b||, so c5 uses the drivers' default 1e-10
    inner_tol = 1e-12 if cfg.n <= 500 else 1e-10
    t0 = time.perf_counter()
    log = (lambda *a: print("[dn] k=%d stokes %d darcy %d dp %.3e dv %.3e t %.1f s" % a, file=sys.stderr, flush=True)) \
        if rank == 0 else None
    if sharded:
        # the subdomain solves split into horizontal strips over the ranks (SDG_DIST_UZAWA / SDG_DIST_AMG)
        from paper_2108_13229_b200 import dist as sd
        drv = drivers.ShardedPartitionedDriver(sc, levels=cfg.v_max_levels, ctx=ctx, inner_tol_rel=inner_tol,
                                               max_coupling_iterations=args.coupling_iterations or 100, log=log,
                                               transport=sd.NcclTransport(ctx))
    else:
        drv = drivers.PartitionedDriver(sc, levels=cfg.v_max_levels, ctx=ctx, inner_tol_rel=inner_tol,
                                        max_coupling_iterations=args.coupling_iterations or 100, log=log)
    print(f"[dn] setup {time.perf_counter() - t0:.1f} s", file=sys.stderr, flush=True)
    setup_s = time.perf_counter() - t0
    n_s, n_d = drv.stokes_matrix.n_rows, drv.darcy_matrix.n_rows
    for _ in range(args.warmup):
        drv.trace_v[:] = 0.0
        drv.trace_p[:] = 0.0
        drv.coupled_step()
    clocks = ClockSampler(local_rank)
    clocks.start()
    launches0 = ctx.launches
    work, solve_s, wall_s, outs = 0.0, 0.0, 0.0, []
    for _ in range(args.steps):
        drv.trace_v[:] = 0.0
        drv.trace_p[:] = 0.0
        out = drv.coupled_step()
        outs.append(out)
        work += n_s * sum(out.stokes_iterations) + n_d * sum(out.darcy_iterations)
        solve_s += out.solve_seconds
        wall_s += out.seconds
    launches = ctx.launches - launches0
    clk = clocks.stop()
    last = outs[-1]
    if world > 1:  # whole-job numbers: the slowest rank's time; sharded: one system, replicas: N systems
        import torch
        import torch.distributed as tdist
        dev = torch.device("cuda", local_rank)
        solve_s, w_sum = job_totals(tdist, solve_s, work, dev)
        wall_s, _ = job_totals(tdist, wall_s, 0.0, dev)
        work = work if sharded else w_sum
    line = {
        "metric": METRIC, "value": work / solve_s, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * wall_s / args.steps, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.n}x{cfg.n} cells per subdomain, partitioned Dirichlet-Neumann "
                               f"(free flow {n_s:,} DoF: PD-GMRES + Uzawa(AMG_V); porous {n_d:,} DoF: BiCGSTAB + "
                               f"AMG), IQN-ILS after a 0.5-relaxed first step, interface measures < 1e-8, "
                               f"inner tol {inner_tol:g}*||b||, AMG levels {cfg.v_max_levels}",
                   "dof": n_s + n_d,
                   "parallelism": (f"subdomain solves over horizontal strips x{world}" if sharded else
                                   "single GPU" if world == 1 else f"replicas x{world}"), "setup_s": setup_s,
                   "coupling_iterations": last.coupling_iterations, "converged": last.converged,
                   "stokes_iterations": last.stokes_iterations, "darcy_iterations": last.darcy_iterations,
                   "measures_p": last.measure_p, "measures_v": last.measure_v,
                   "l2": "matrix and vectors exceed the 126 MB L2" if n_s > 4_000_000 else "not flushed"},
        "gpu_launches": launches, "clocks": clk,
        "e2e": {"value": work / wall_s, "unit": UNIT, "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                "ms_per_step": 1e3 * wall_s / args.steps,
                "timing": "host wall clock of the whole coupling loop (every subdomain solve is a host-pointer "
                          "C-ABI call: H2D of b, D2H of x inside)"},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1 or sharded:
        import torch.distributed as tdist
        if tdist.is_initialized():
            tdist.destroy_process_group()
    return 0


def run_sharded(args):
    """One system split into horizontal strips over the ranks,
    NCCL transport; `value` = DoF*iterations of the whole system / max-over-ranks
    device time (strong scaling: the work is fixed as N grows)."""
    import torch
    rank, local_rank, world = dist_env()
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    from paper_2108_13229_b200 import dist as sd
    from paper_2108_13229_b200 import scenarios, sdc

    cfg = scenarios.CONFIGS[args.config]
    s = scenarios.build_system(cfg)
    n = s.n_total()
    tol = 1e-8 * float(np.linalg.norm(s.rhs))
    ctx = sdc.Context(local_rank)
    tr = sd.NcclTransport(ctx)
    ds = sd.DistSystem(s, tr, ctx=ctx)
    t0 = time.perf_counter()
    p = sd.DistTdPreconditioner(ds, "td_bgs", cfg.v_max_levels, cfg.d_max_levels)
    setup_s = time.perf_counter() - t0
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    b_loc = ds.local(s.rhs)
    b_dev = torch.from_numpy(b_loc).to(dev)
    x_dev = torch.zeros(ds.n_local(), dtype=torch.float64, device=dev)
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    ctrl = sdc.RestartController.fixed(50) if cfg.solver == "gmres50" else sdc.RestartController.defaults()
    max_it = 20000 if cfg.solver == "bicgstab" else 4000

    def step():
        return sd.dist_solve_device(ds, p, cfg.solver, b_dev.data_ptr(), x_dev.data_ptr(), tol, max_it, ctrl)

    torch.cuda.synchronize()
    for _ in range(args.warmup):
        rep = step()
    clocks = ClockSampler(local_rank)
    clocks.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    evs, iters = [], []
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        rep = step()
        with torch.cuda.stream(stream):
            e1.record(stream)
        evs.append((e0, e1))
        iters.append(rep.iterations)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches = ctx.launches - launches0
    clk = clocks.stop()
    total_ms = sum(a.elapsed_time(b) for a, b in evs)
    # strong scaling: every rank reports the same iterations of the one system
    total_ms, _ = job_totals(dist, total_ms, 0.0, dev)
    value = float(n) * sum(iters) / (total_ms / 1e3)
    e2e = None
    if not args.no_e2e:
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        e_its = 0
        for _ in range(args.steps):
            res = (sd.dist_bicgstab(ds, p, b_loc, tol, max_it) if cfg.solver == "bicgstab"
                   else sd.dist_pd_gmres(ds, p, b_loc, tol, max_it, ctrl))
            e_its += res.report.iterations
        e_s = time.perf_counter() - t0
        e_s, _ = job_totals(dist, e_s, 0.0, dev)
        e2e = {"value": float(n) * e_its / e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * ds.n_local(),
               "d2h_bytes_per_step": 8 * ds.n_local(), "ms_per_step": 1e3 * e_s / args.steps,
               "timing": "host wall clock around the synchronous sdg_dist_* call, max over ranks"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_for(cfg, n, s.matrix.nnz(), args),
        "details": {"iterations": iters, "setup_s": setup_s, "omega": p.omega(), "local_rows": ds.n_local()},
        "gpu_launches": launches, "clocks": clk, "e2e": e2e,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def launcher_cmd(args, port):
    """`bench.py --gpus N` without a rank environment re-launches itself as N
    ranks, the way the driver does (torch.distributed.run, one process per
    GPU, rendezvous on 127.0.0.1)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        return subprocess.call(launcher_cmd(args, port))
    if args.impl == "reference":
        return run_reference(args)
    from paper_2108_13229_b200 import scenarios
    if scenarios.CONFIGS[args.config].solver == "dn":
        return run_partitioned(args)
    if args.sharded or (dist_env()[2] > 1 and not args.replicas):
        return run_sharded(args)
    if scenarios.CONFIGS[args.config].steps > 1:
        return run_transient(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
