"""Dev probe: preconditioner-apply parity and BiCGSTAB counts of one config
against the reference (python scripts/probe_cfg.py c4s)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2108_13229_b200 import scenarios, sdc
from oracle.refpy import RefLib, Csr, System
cfg = scenarios.CONFIGS[sys.argv[1]]
t = cfg.dt if cfg.steps > 1 else None
s = scenarios.build_system(cfg, t=t)
n = s.n_total()
R = RefLib()
rs = System(n, s.n_u, s.n_vel, s.n_pff, s.n_ppm, Csr(n, n, s.matrix.row_offsets, s.matrix.col_indices, s.matrix.values), s.rhs)
td = R.td(rs, "td_bgs", cfg.v_max_levels, cfg.d_max_levels)
p = sdc.TdPreconditioner(s, "td_bgs", cfg.v_max_levels, cfg.d_max_levels)
print("omega gpu", p.omega(), "hier", p.hierarchy(0), p.hierarchy(1), flush=True)
r = np.random.default_rng(1).standard_normal(n)
zg = p.apply(r)
zr = R.td_apply(td, r) if hasattr(R, "td_apply") else td.apply(r)
print("apply rel diff", np.linalg.norm(zg - zr) / np.linalg.norm(zr), flush=True)
for blk, (a, b) in {"v": (0, s.n_vel), "pff": (s.n_vel, s.n_vel + s.n_pff), "pm": (s.n_vel + s.n_pff, n)}.items():
    print("  block", blk, np.linalg.norm(zg[a:b] - zr[a:b]) / max(np.linalg.norm(zr[a:b]), 1e-300), flush=True)
tol = 1e-8 * np.linalg.norm(s.rhs)
t0 = time.time()
res = sdc.bicgstab(s.matrix, p, s.rhs, tol, 20000)
print("gpu bicgstab", res.report.iterations, res.report.converged, time.time() - t0, flush=True)
