"""Generates tests/golden/c4s_reference.json: BASELINE config 4's transient
(implicit Euler dt = 0.1 x 10, log-normal K, warm-started BiCGSTAB + td_bgs,
AMG L4) at 250^2 by the compiled reference (oracle/_ref): per time step the
iteration count and size-independent fingerprints of x (||x||, dot products
with seeded random vectors, a strided sample), plus the reference's own
iteration-count spread under legal rounding changes (the ensemble of
scripts/ref_spread_c4.py: -O2 and FMA builds, right-hand sides perturbed by
one ulp; profiles/r02/ref_spread_c4s.jsonl).  Checker-side script."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.refpy import Csr, RefLib, System  # noqa: E402
from paper_2108_13229_b200 import scenarios  # noqa: E402

cfg = scenarios.CONFIGS["c4s"]
OUT = os.path.join(ROOT, "tests", "golden", "c4s_reference.json")
ENSEMBLE_ONLY = "--ensemble-only" in sys.argv  # refresh the spread from the jsonl, keep the step fingerprints
R = None if ENSEMBLE_ONLY else RefLib()
x, td, a = None, None, None
steps = json.load(open(OUT))["steps"] if ENSEMBLE_ONLY else []
n = cfg.dof
t0 = time.time()
for k in range(1, 0 if ENSEMBLE_ONLY else cfg.steps + 1):
    v_prev = None if x is None else x[: 2 * cfg.n * (cfg.n + 1)]
    s = scenarios.build_system(cfg, t=k * cfg.dt, v_prev=v_prev)
    n = s.n_total()
    if td is None:
        a = Csr(n, n, s.matrix.row_offsets, s.matrix.col_indices, s.matrix.values)
        td = R.td(System(n, s.n_u, s.n_vel, s.n_pff, s.n_ppm, a, s.rhs), "td_bgs", cfg.v_max_levels,
                  cfg.d_max_levels)
    tol = 1e-8 * np.linalg.norm(s.rhs)
    if x is None:
        x, rep = R.bicgstab(a, s.rhs, tol, 20000, precond=td)
    else:
        d, rep = R.bicgstab(a, R.spmv_add(a, x, s.rhs, -1.0), tol, 20000, precond=td)
        x = x + d
    rng = np.random.default_rng(1000 + k)
    probes = rng.standard_normal((4, n))
    steps.append({"step": k, "iterations": int(rep.iterations), "x_norm": float(np.linalg.norm(x)),
                  "dots": [float(v) for v in probes @ x], "sample_stride": 997,
                  "sample": [float(v) for v in x[::997]]})
    print(k, rep.iterations, time.time() - t0, flush=True)
ens = [json.loads(l) for l in open(os.path.join(ROOT, "profiles", "r02", "ref_spread_c4s.jsonl"))]
its = np.array([e["iterations"] for e in ens if len(e["iterations"]) == cfg.steps])
out = {"config": "c4s", "n": cfg.n, "dof": int(n), "steps": steps,
       "ensemble": {"runs": len(its), "min": its.min(0).tolist(), "max": its.max(0).tolist(),
                    "median": np.median(its, 0).tolist(), "totals": its.sum(1).tolist(),
                    "source": "profiles/r02/ref_spread_c4s.jsonl (scripts/ref_spread_c4.py)"}}
with open(OUT, "w") as f:
    json.dump(out, f, indent=1)
