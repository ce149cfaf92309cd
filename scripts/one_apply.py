"""Dev aid: a few td_bgs (or AMG V / D) applies of a config, for ncu launch lists:
python scripts/one_apply.py c3 td|V|D [applies]"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2108_13229_b200 import scenarios, sdc
cfg = scenarios.CONFIGS[sys.argv[1]]
which = sys.argv[2] if len(sys.argv) > 2 else "td"
k = int(sys.argv[3]) if len(sys.argv) > 3 else 2
s = scenarios.build_system(cfg)
if which == "td":
    p = sdc.TdPreconditioner(s, "td_bgs", cfg.v_max_levels, cfg.d_max_levels)
    n = s.n_total()
elif which == "V":
    mat = sdc.submatrix(s.matrix, 0, s.n_vel, 0, s.n_vel)
    p = sdc.AmgPreconditioner(mat, sdc.AmgOptions(components=[0] * s.n_u + [1] * (s.n_vel - s.n_u),
                                                  max_levels=cfg.v_max_levels))
    n = mat.n_rows
else:
    mat = sdc.ground_dof(sdc.submatrix(s.matrix, s.n_vel + s.n_pff, s.n_total(), s.n_vel + s.n_pff, s.n_total()))
    p = sdc.AmgPreconditioner(mat, sdc.AmgOptions(max_levels=cfg.d_max_levels))
    n = mat.n_rows
r = np.random.default_rng(1).standard_normal(n)
for _ in range(k):
    p.apply(r)
print("done")
