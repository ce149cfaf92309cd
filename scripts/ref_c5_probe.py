"""Checker-side probe: the first coupling iterations of the partitioned
Dirichlet-Neumann loop of BASELINE config 5, composed from the unmodified
reference's own pieces (assemble_stokes / assemble_darcy with interface data,
UzawaPreconditioner(AMG) + PD-GMRES defaults for the free flow, AMG + BiCGSTAB
for the porous medium, its traces; coupling.cpp:148-242, 252-332), with the
stop rule of bench.py's config-5 driver (inner tol 1e-12 ||b||).  Writes one
JSON line per coupling iteration and the interface traces (npz) to compare the
GPU driver's first iterations with (tests/test_gpu_partitioned.py).

    python scripts/ref_c5_probe.py n K levels iterations out_prefix
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle.refpy import RefLib
from paper_2108_13229_b200.iqn import IqnIlsHistory, iqn_ils_update

n, K, lv, iters, out = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
tol_rel = 1e-12
R = RefLib()
t0 = time.time()
A_s, _ = R.stokes(n, permeability=K, v_gamma=np.zeros(n))
uz = R.uzawa_stokes(A_s, n, lv)
D, _ = R.darcy(n, K, np.zeros(n))
amg = R.amg_precond(D, lv)
print(json.dumps({"n": n, "K": K, "levels": lv, "setup_s": time.time() - t0}), flush=True)
v, p_k = np.zeros(n), np.zeros(n)
hist = IqnIlsHistory()
traces = {}
for k in range(iters):
    t1 = time.time()
    _, b = R.stokes(n, permeability=K, v_gamma=v)
    x, rep = R.pd_gmres(A_s, b, tol_rel * np.linalg.norm(b), 400, precond=uz)
    pt = R.stokes_pressure_trace(n, 1.0, x)
    _, db = R.darcy(n, K, pt)
    p, rep2 = R.bicgstab(D, db, tol_rel * np.linalg.norm(db), 10000, precond=amg)
    vt = R.darcy_velocity_trace(n, K, p, pt)
    dp, npn = np.linalg.norm(pt - p_k), np.linalg.norm(pt)
    dv, nv = np.linalg.norm(vt - v), np.linalg.norm(vt)
    print(json.dumps({"k": k, "stokes_iterations": rep.iterations, "stokes_converged": rep.converged,
                      "darcy_iterations": rep2.iterations, "darcy_converged": rep2.converged,
                      "measure_p": dp / max(npn, 1e-300), "measure_v": dv / max(nv, 1e-300),
                      "seconds": time.time() - t1}), flush=True)
    traces[f"p_{k}"], traces[f"v_{k}"] = pt, vt
    np.savez(out + "_traces.npz", **traces)
    res = vt - v
    if not hist.has_previous():
        v = v + 0.5 * res
        hist.record(res, vt)
    else:
        v = iqn_ils_update(hist, v, res, vt)
    p_k = pt
