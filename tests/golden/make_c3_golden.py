"""Generates tests/golden/c3_reference.json: the reference's own GMRES(50) +
td_bgs solve of BASELINE config 3 (500^2, K=1e-2, AMG L3; ~10 min on one core,
most of it the reference's coarse lu_factor), reduced to size-independent
fingerprints the GPU test can check: iteration count, ||x||, a strided sample
of x, and dot products with seeded random vectors.  Checker-side script (runs
the compiled reference from oracle/_ref)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.refpy import Csr, RefLib, System  # noqa: E402
from paper_2108_13229_b200 import scenarios  # noqa: E402

cfg = scenarios.CONFIGS["c3"]
s = scenarios.build_system(cfg)
n = s.n_total()
R = RefLib()
rs = System(n, s.n_u, s.n_vel, s.n_pff, s.n_ppm, Csr(n, n, s.matrix.row_offsets, s.matrix.col_indices,
                                                    s.matrix.values), s.rhs)
t0 = time.time()
td = R.td(rs, "td_bgs", cfg.v_max_levels, cfg.d_max_levels)
setup = time.time() - t0
tol = 1e-8 * float(np.linalg.norm(s.rhs))
t0 = time.time()
x, rep = R.pd_gmres(rs.a, s.rhs, tol, 4000, precond=td, m_init=50, m_min=50, m_max=50)
solve = time.time() - t0
probes = [np.random.default_rng(seed).standard_normal(n) for seed in (1, 2, 3)]
out = {"config": "c3", "n_total": n, "iterations": rep.iterations, "converged": bool(rep.converged),
       "final_residual": rep.final_residual, "tol": tol, "x_norm": float(np.linalg.norm(x)),
       "stride": 997, "x_sample": x[::997].tolist(), "probe_seeds": [1, 2, 3],
       "probe_dots": [float(np.dot(p, x)) for p in probes], "reference_setup_s": setup, "reference_solve_s": solve}
with open(os.path.join(ROOT, "tests", "golden", "c3_reference.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "x_sample"}))
