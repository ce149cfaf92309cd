"""Checker-side probe: how long the unmodified reference takes on c3 (500^2,
K=1e-2, td_bgs with 3 AMG levels) on this host: its own assembly, its setup
(amg_setup + lu_factor of the coarsest level + power iteration), and one
GMRES(50) restart cycle (the reference arm's per-step sample in bench.py)."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.refpy import RefLib  # noqa: E402
R = RefLib()
t0 = time.perf_counter()
rs = R.assemble(500, permeability=1e-2)
t_asm = time.perf_counter() - t0
t0 = time.perf_counter()
td = R.td(rs, "td_bgs", 3, 3)
t_setup = time.perf_counter() - t0
print(json.dumps({"assembly_s": t_asm, "setup_s": t_setup}), flush=True)
tol = 1e-8 * np.linalg.norm(rs.rhs)
for _ in range(2):
    t0 = time.perf_counter()
    _, rep = R.pd_gmres(rs.a, rs.rhs, tol, 1, precond=td, m_init=50, m_min=50, m_max=50)
    dt = time.perf_counter() - t0
    print(json.dumps({"cycle_s": dt, "iterations": rep.iterations, "dof_it_s": rs.n * rep.iterations / dt}), flush=True)
