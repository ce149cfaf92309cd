"""Dev aid: AMG V-cycle with the lattice smoother vs without (knob on one
matrix size); prints where they differ.  python scripts/lat_debug.py c1 split|default"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2108_13229_b200 import scenarios, sdc
cfg = scenarios.CONFIGS[sys.argv[1]]
mode = sys.argv[2] if len(sys.argv) > 2 else "default"
os.environ["SDG_DEBUG"] = "1"
s = scenarios.build_system(cfg)
V = sdc.submatrix(s.matrix, 0, s.n_vel, 0, s.n_vel)
opts = sdc.AmgOptions(components=[0] * s.n_u + [1] * (s.n_vel - s.n_u), max_levels=cfg.v_max_levels)
if mode == "split":
    os.environ["SDG_GS_SPLIT"] = "1"
r = np.random.default_rng(0).standard_normal(V.n_rows)
a = sdc.AmgPreconditioner(V, opts)
print("features", a.features(), a.hierarchy(), flush=True)
za = a.apply(r)
za2 = a.apply(r)
os.environ["SDG_GS_LATTICE"] = "0"
b = sdc.AmgPreconditioner(V, opts)
zb = b.apply(r)
d = np.abs(za - zb)
print("repeat equal", np.array_equal(za, za2), "max diff", d.max(), "rel", np.linalg.norm(za - zb) / np.linalg.norm(zb))
idx = np.where(d > 1e-12 * np.abs(zb).max())[0]
print("n differing", idx.size, "first", idx[:20], "u/v split at", s.n_u)
