"""Dev: per-warp clock64 spans of the 5-point chain kernel (SDG_CHAIN_MODE=8) on
the finest Darcy level of a config."""
import os, sys, ctypes as C
import numpy as np
sys.path.insert(0, os.getcwd())
os.environ.setdefault("SDG_CHAIN_MODE", "8")
import torch
from paper_2108_13229_b200 import scenarios, sdc
cfg = scenarios.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
s = scenarios.build_system(cfg)
nff = s.n_vel + s.n_pff
D = sdc.ground_dof(sdc.submatrix(s.matrix, nff, s.n_total(), nff, s.n_total()), 0)
n = D.n_rows
# a one-level-above-coarse AMG on D: level 0 uses the chain smoother; sor_sweep path is the bitwise kernel,
# so drive the chain through an AMG apply and read the clock slots appended past z (z is the level's output).
# Simplest: use the AMG preconditioner with 2 levels and an oversized output buffer via the device API.
p = sdc.AmgPreconditioner(D, sdc.AmgOptions(max_levels=2))
r = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
z = torch.zeros(n + 64, dtype=torch.float64, device="cuda")
for _ in range(3):
    sdc.lib().sdg_precond_apply_device(p.h, C.c_void_p(r.data_ptr()), C.c_void_p(z.data_ptr()))
torch.cuda.synchronize()
t = z[n:n + 16].cpu().numpy()
nb = int((int(np.sqrt(n)) + 31) // 32)
t0 = t[0]
for w in range(nb):
    print(f"warp {w}: start {t[2*w]-t0:9.0f} end {t[2*w+1]-t0:9.0f} span {t[2*w+1]-t[2*w]:9.0f}")
