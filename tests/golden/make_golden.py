"""Regenerate tests/golden/*.npz from the reference itself.

Runs the UNMODIFIED reference library (oracle/_ref/libsdcore_ref.so, built by
`make -C oracle ref` from /root/reference) and stores small input/output
vectors, so the GPU box -- where /root/reference does not exist -- can check
against the reference's own outputs.  Usage:

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.refpy import RefLib  # noqa: E402


def csr(prefix, a):
    return {f"{prefix}_rowptr": a.rowptr, f"{prefix}_col": a.col, f"{prefix}_val": a.val}


def system_case(R: RefLib, n: int, permeability: float, name: str, solvers=("gmres50", "pdgmres", "bicgstab")):
    s = R.assemble(n, permeability=permeability)
    td = R.td(s, "td_bgs")
    out = {"n": n, "permeability": permeability, "n_total": s.n, "n_u": s.n_u, "n_vel": s.n_vel,
           "n_pff": s.n_pff, "n_ppm": s.n_ppm, "rhs": s.rhs, "omega": td.omega}
    out.update(csr("A", s.a))
    r = R.random_vector(s.n, 17)
    out["apply_r"] = r
    out["apply_z"] = td.apply(r)
    tol = 1e-8 * np.linalg.norm(s.rhs)
    out["tol"] = tol
    for solver in solvers:
        if solver == "gmres50":
            x, rep = R.pd_gmres(s.a, s.rhs, tol, 400, precond=td, m_init=50, m_min=50, m_max=50)
        elif solver == "pdgmres":
            x, rep = R.pd_gmres(s.a, s.rhs, tol, 400, precond=td)
        else:
            x, rep = R.bicgstab(s.a, s.rhs, tol, 20000, precond=td)
        out[f"{solver}_x"] = x
        out[f"{solver}_iters"] = rep.iterations
        out[f"{solver}_hist"] = rep.residual_history
    vh = td.v_hierarchy
    for lev, L in enumerate(vh.levels()):
        if L.aggregate_of is not None:
            out[f"vagg{lev}"] = L.aggregate_of
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, {k: out[k] for k in out if k.endswith("_iters")}, "omega", out["omega"])


def dominant_case(R: RefLib):
    out = {}
    for seed in (3, 14):
        a = R.random_dominant(100, 0.08, seed)
        b = R.random_vector(100, seed + 50)
        tol = 1e-12 * np.linalg.norm(b)
        out.update(csr(f"A{seed}", a))
        out[f"b{seed}"] = b
        out[f"xlu{seed}"] = R.lu_solve(a, b)
        x, rep = R.pd_gmres(a, b, tol, 200)
        out[f"xg{seed}"], out[f"ig{seed}"] = x, rep.iterations
        x, rep = R.bicgstab(a, b, tol, 500)
        out[f"xb{seed}"], out[f"ib{seed}"] = x, rep.iterations
        z0 = R.random_vector(100, seed + 7)
        out[f"gs_z0_{seed}"] = z0
        out[f"gs_z1_{seed}"] = R.sor_sweep(a, z0, b, 1.0)
        out[f"gs_z1w_{seed}"] = R.sor_sweep(a, z0, b, 0.7)
        out[f"spmv_{seed}"] = R.spmv(a, z0)
        h = R.amg_setup(a, coarse_threshold=10)
        out[f"vcyc_{seed}"] = h.vcycle(b)
        out[f"vcyc_levels_{seed}"] = h.num_levels
    np.savez_compressed(os.path.join(HERE, "dominant.npz"), **out)
    print("dominant", {k: int(out[k]) for k in out if k.startswith(("ig", "ib"))})


def main():
    R = RefLib()
    system_case(R, 6, 1.0, "system_n6")
    system_case(R, 16, 1e-2, "system_n16")
    system_case(R, 50, 1.0, "system_c1")
    dominant_case(R)


if __name__ == "__main__":
    main()
