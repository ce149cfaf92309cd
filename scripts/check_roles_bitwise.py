"""Dev check: AMG V-cycles over the c3 velocity block and porous block with
the walk roles on and off must agree bitwise (several applies each)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2108_13229_b200 import scenarios, sdc
cfg = scenarios.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
s = scenarios.build_system(cfg)
A = s.matrix
V = sdc.submatrix(A, 0, s.n_vel, 0, s.n_vel)
D = sdc.ground_dof(sdc.submatrix(A, s.n_vel + s.n_pff, s.n_total(), s.n_vel + s.n_pff, s.n_total()))
comps = [0] * s.n_u + [1] * (s.n_vel - s.n_u)
rng = np.random.default_rng(3)
ok = True
for name, M, opts in (("V", V, sdc.AmgOptions(components=comps, max_levels=cfg.v_max_levels)),
                      ("D", D, sdc.AmgOptions(max_levels=cfg.d_max_levels))):
    xs = [rng.standard_normal(M.n_rows) for _ in range(3)]
    out = {}
    for roles in ("1", "0"):
        os.environ["SDG_WALK_ROLES"] = roles
        p = sdc.AmgPreconditioner(M, opts)
        out[roles] = [p.apply(x) for x in xs] + [p.apply(xs[0])]
    same = all(np.array_equal(a, b) for a, b in zip(out["1"], out["0"]))
    rep = np.array_equal(out["1"][0], out["1"][3])
    diff = max(float(np.max(np.abs(a - b)) / np.max(np.abs(b))) for a, b in zip(out["1"], out["0"]))
    print(name, M.n_rows, "roles==plain", same, "repeatable", rep, "max rel diff", diff)
    ok = ok and same and rep
print("OK" if ok else "MISMATCH")
