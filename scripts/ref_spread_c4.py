"""Checker-side probe: the reference's own BiCGSTAB iteration-count spread on
the config-4 transient (c4s: 250^2, log-normal K, L4, 10 implicit-Euler steps,
warm-started), under legal rounding changes:

  * build: the unmodified reference at -O2 (its Release build) and the same
    sources with FMA contraction (oracle/Makefile ref_fma);
  * rhs perturbation: every step's right-hand side multiplied element-wise by
    (1 + 2^-52 u), u ~ U(-1, 1) from a seeded generator -- a rounding-level
    change of the input, the size of the differences a reassociated GPU
    kernel introduces per operation.

One JSON line per variant with the per-step iteration counts.  The GPU test
bounds (tests/test_gpu_transient.py) come from this spread.

    python scripts/ref_spread_c4.py <build: O2|fma> <seed: -1 = unperturbed> [config]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.refpy import REF_SO, Csr, RefLib, System  # noqa: E402
from paper_2108_13229_b200 import scenarios  # noqa: E402

build, seed = sys.argv[1], int(sys.argv[2])
cfg = scenarios.CONFIGS[sys.argv[3] if len(sys.argv) > 3 else "c4s"]
steps = int(sys.argv[4]) if len(sys.argv) > 4 else cfg.steps
so = REF_SO if build == "O2" else REF_SO.replace("libsdcore_ref.so", "libsdcore_ref_fma.so")
R = RefLib(so)
rng = np.random.default_rng(seed) if seed >= 0 else None
x, td, a = None, None, None
its, t0 = [], time.time()
status = "ok"
for k in range(1, steps + 1):
    t = k * cfg.dt if cfg.steps > 1 else None
    v_prev = None if x is None else x[: 2 * cfg.n * (cfg.n + 1)]
    s = scenarios.build_system(cfg, t=t, v_prev=v_prev)
    n = s.n_total()
    rhs = s.rhs.copy()
    if rng is not None:
        rhs *= 1.0 + np.ldexp(rng.uniform(-1.0, 1.0, n), -52)
    if td is None:
        a = Csr(n, n, s.matrix.row_offsets, s.matrix.col_indices, s.matrix.values)
        td = R.td(System(n, s.n_u, s.n_vel, s.n_pff, s.n_ppm, a, rhs), "td_bgs", cfg.v_max_levels,
                  cfg.d_max_levels)
    tol = 1e-8 * np.linalg.norm(rhs)
    try:
        if x is None:
            x, rep = R.bicgstab(a, rhs, tol, 20000, precond=td)
        else:
            d, rep = R.bicgstab(a, R.spmv_add(a, x, rhs, -1.0), tol, 20000, precond=td)
            x = x + d
    except Exception as e:  # the reference throws on a repeated breakdown (krylov.cpp:213-221)
        status = f"step {k}: {e}"
        break
    its.append(int(rep.iterations))
print(json.dumps({"config": cfg.name, "build": build, "seed": seed, "iterations": its, "total": sum(its),
                  "status": status, "seconds": round(time.time() - t0, 1)}), flush=True)
