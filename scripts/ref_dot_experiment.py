"""Checker-side experiment: how much of the reference's BiCGSTAB iteration-count
spread on the config-4 transient (c4s) comes from the rounding error of its dot
products.  Runs the C restatement of the reference (oracle/sdc_oracle.c, pinned
bitwise to the compiled reference) on the reference's own preconditioner
hierarchies, once with the reference's sequential dot and once with pairwise
summation (the error behaviour of a GPU tree reduction).

    python scripts/ref_dot_experiment.py <mode: 0 sequential | 1 pairwise> [config]
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.refpy import Csr, OHier, PortLib, RefLib, System  # noqa: E402
from paper_2108_13229_b200 import scenarios  # noqa: E402

mode = int(sys.argv[1])
cfg = scenarios.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c4s"]
R, port = RefLib(), PortLib()
port.L.orc_set_dot_mode.argtypes = [C.c_int]
port.L.orc_set_dot_mode.restype = None
port.L.orc_set_dot_mode(mode)
x, bundle, a = None, None, None
its, t0 = [], time.time()
for k in range(1, cfg.steps + 1):
    v_prev = None if x is None else x[: 2 * cfg.n * (cfg.n + 1)]
    s = scenarios.build_system(cfg, t=k * cfg.dt, v_prev=v_prev)
    n = s.n_total()
    if bundle is None:
        a = Csr(n, n, s.matrix.row_offsets, s.matrix.col_indices, s.matrix.values)
        td = R.td(System(n, s.n_u, s.n_vel, s.n_pff, s.n_ppm, a, s.rhs), "td_bgs", cfg.v_max_levels, cfg.d_max_levels)
        vh, dh = OHier.from_ref(td.v_hierarchy), OHier.from_ref(td.d_hierarchy)
        A = sp.csr_matrix((a.val, a.col, a.rowptr), shape=(n, n))

        def sub(rb, re, cb, ce):
            m = A[rb:re, cb:ce].tocsr()
            m.sort_indices()
            return Csr(m.shape[0], m.shape[1], m.indptr.astype(np.int32), m.indices.astype(np.int32), m.data)

        n_ff = s.n_vel + s.n_pff
        bundle = port.td_bundle(vh, sub(s.n_vel, n_ff, 0, s.n_vel), td.omega, sub(n_ff, n, 0, n_ff), dh, s.n_vel,
                                s.n_pff, s.n_ppm)
    tol = 1e-8 * np.linalg.norm(s.rhs)
    if x is None:
        x, rep = port.bicgstab(a, s.rhs, tol, 20000, precond=bundle)
    else:
        d, rep = port.bicgstab(a, s.rhs - A @ x, tol, 20000, precond=bundle)
        x = x + d
    its.append(int(rep.iterations))
    print(k, rep.iterations, round(time.time() - t0, 1), file=sys.stderr, flush=True)
print(json.dumps({"config": cfg.name, "dot": "pairwise" if mode else "sequential", "iterations": its, "total": sum(its),
                  "seconds": round(time.time() - t0, 1)}), flush=True)
