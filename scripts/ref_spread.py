"""Checker-side probe: the reference's own iteration-count spread under a
legal rounding change (FMA contraction), on the bench systems.  Runs the
unmodified reference (oracle/_ref/libsdcore_ref.so, -O2 as its Release build)
and the same sources compiled with -mfma -ffp-contract=fast
(libsdcore_ref_fma.so), prints one JSON line per (config, solver, build)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.refpy import REF_SO, Csr, RefLib, System  # noqa: E402
from paper_2108_13229_b200 import scenarios  # noqa: E402

configs = sys.argv[1:] or ["c2", "c2u"]
libs = {"ref_O2": RefLib(REF_SO), "ref_fma": RefLib(REF_SO.replace("libsdcore_ref.so", "libsdcore_ref_fma.so"))}
for name in configs:
    cfg = scenarios.CONFIGS[name]
    s = scenarios.build_system(cfg)
    n = s.n_total()
    tol = 1e-8 * np.linalg.norm(s.rhs)
    xs = {}
    for lname, ref in libs.items():
        rs = System(n, s.n_u, s.n_vel, s.n_pff, s.n_ppm,
                    Csr(n, n, s.matrix.row_offsets, s.matrix.col_indices, s.matrix.values), s.rhs)
        td = ref.td(rs, v_max_levels=cfg.v_max_levels, d_max_levels=cfg.d_max_levels) if hasattr(ref, "td") else None
        for solver in ("bicgstab", "gmres50"):
            if solver == "bicgstab":
                x, rep = ref.bicgstab(rs.a, s.rhs, tol, 20000, precond=td)
            else:
                x, rep = ref.pd_gmres(rs.a, s.rhs, tol, 400, precond=td, m_init=50, m_min=50, m_max=50)
            xs[(lname, solver)] = x
            print(json.dumps({"config": name, "build": lname, "solver": solver, "iterations": rep.iterations,
                              "converged": bool(rep.converged)}), flush=True)
    for solver in ("bicgstab", "gmres50"):
        a, b = xs[("ref_O2", solver)], xs[("ref_fma", solver)]
        print(json.dumps({"config": name, "solver": solver,
                          "x_rel_l2_O2_vs_fma": float(np.linalg.norm(a - b) / np.linalg.norm(a))}))
