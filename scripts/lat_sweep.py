"""Dev aid: the lattice lower solve on the GPU vs its host emulation for the
label blocks / levels of a config that are lattices.  python scripts/lat_sweep.py c1"""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import scipy.sparse as sp
from paper_2108_13229_b200 import scenarios, sdc
L = sdc.lib()
ctx = sdc.default_context()
def sub(A, lo, hi):
    M = sp.csr_matrix((A.values, A.col_indices, A.row_offsets), shape=(A.n_rows, A.n_rows))[lo:hi, lo:hi].tocsr()
    M.sort_indices()
    return sdc.SparseMatrix(hi - lo, hi - lo, M.indptr.astype(np.int32), M.indices.astype(np.int32), M.data)
def run(name, A, reps=1):
    n = A.n_rows
    b = np.random.default_rng(0).standard_normal(n)
    zh, zd = np.zeros(n), np.zeros(n)
    P = C.c_void_p
    rp, ci, v = (np.ascontiguousarray(A.row_offsets, np.int32), np.ascontiguousarray(A.col_indices, np.int32),
                 np.ascontiguousarray(A.values))
    rc = L.sdg_debug_lattice_sweep(ctx.h, n, rp.ctypes.data_as(P), ci.ctypes.data_as(P), v.ctypes.data_as(P),
                                   b.ctypes.data_as(P), zh.ctypes.data_as(P), zd.ctypes.data_as(P), reps)
    if rc != 0:
        print(name, n, "not a lattice"); return
    d = np.abs(zh - zd)
    bad = np.where(d > 0)[0]
    print(name, n, "reps", reps, "bitwise" if bad.size == 0 else f"DIFF {bad.size} first {bad[:10]} max {d.max():.3e}", flush=True)
for cname in sys.argv[1:]:
    cfg = scenarios.CONFIGS[cname]
    s = scenarios.build_system(cfg)
    V = sdc.submatrix(s.matrix, 0, s.n_vel, 0, s.n_vel)
    hv = sdc.host_hierarchy(V, sdc.AmgOptions(components=[0] * s.n_u + [1] * (s.n_vel - s.n_u), max_levels=cfg.v_max_levels))
    nu1 = hv[0].aggregate_of[:s.n_u].max() + 1
    D = sdc.ground_dof(sdc.submatrix(s.matrix, s.n_vel + s.n_pff, s.n_total(), s.n_vel + s.n_pff, s.n_total()))
    hd = sdc.host_hierarchy(D, sdc.AmgOptions(max_levels=cfg.d_max_levels))
    for reps in (1, 2, 3):
        run(cname + " V0u", sub(V, 0, s.n_u), reps)
        run(cname + " V1v", sub(hv[1].a, nu1, hv[1].a.n_rows), reps)
        run(cname + " V1u", sub(hv[1].a, 0, nu1), reps)
        run(cname + " D0", D, reps)
        run(cname + " D1", hd[1].a, reps)
