"""Checker-side probe: the partitioned Dirichlet-Neumann loop composed from the
reference's own pieces (assemble_stokes/darcy, Uzawa/AMG, pd_gmres/bicgstab,
traces, IQN-ILS), printing per coupling iteration the inner iteration counts
and the two relative interface measures.  usage: ref_dn_probe.py n K [levels]"""
import sys, time; import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle.refpy import RefLib
from paper_2108_13229_b200.iqn import IqnIlsHistory, iqn_ils_update
R = RefLib()
n = int(sys.argv[1]); K = float(sys.argv[2]); lv = int(sys.argv[3]) if len(sys.argv) > 3 else 3
A_s, _ = R.stokes(n, permeability=K, v_gamma=np.zeros(n))
uz = R.uzawa_stokes(A_s, n, lv)
D, _ = R.darcy(n, K, np.zeros(n))
amg = R.amg_precond(D, lv)
v = np.zeros(n); p_k = np.zeros(n)
hist = IqnIlsHistory()
t0 = time.time()
for k in range(100):
    _, b = R.stokes(n, permeability=K, v_gamma=v)
    x, rep = R.pd_gmres(A_s, b, 1e-10 * np.linalg.norm(b), 400, precond=uz)
    pt = R.stokes_pressure_trace(n, 1.0, x)
    _, db = R.darcy(n, K, pt)
    p, rep2 = R.bicgstab(D, db, 1e-10 * np.linalg.norm(db), 10000, precond=amg)
    vt = R.darcy_velocity_trace(n, K, p, pt)
    dp, npn = np.linalg.norm(pt - p_k), np.linalg.norm(pt); dv, nv = np.linalg.norm(vt - v), np.linalg.norm(vt)
    print(k, rep.iterations, rep2.iterations, dp / max(npn, 1e-300), dv / max(nv, 1e-300), flush=True)
    if dp < 1e-8 * npn and dv < 1e-8 * nv: print("converged", k + 1, time.time() - t0); break
    res = vt - v
    if not hist.has_previous():
        v = v + 0.5 * res; hist.record(res, vt)
    else:
        v = iqn_ils_update(hist, v, res, vt)
    p_k = pt
