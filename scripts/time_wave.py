"""Dev helper: device time of N AMG V-cycle applies of the velocity block
(MAC) and of the porous block (5-point) of one config, each alone on the
stream, for the default plans and with the multi-SM smoothers switched off
level by level (SDG_GS_WAVE=0 on the finest level; the opt-in SDG_GS_LATTICE=1 on level 1).
python scripts/time_wave.py c3 [N]"""
import os, sys, time
import ctypes as C
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2108_13229_b200 import scenarios, sdc
cfg = scenarios.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
n_app = int(sys.argv[2]) if len(sys.argv) > 2 else 50
s = scenarios.build_system(cfg)
ctx = sdc.default_context()
L = sdc.lib()
V = sdc.submatrix(s.matrix, 0, s.n_vel, 0, s.n_vel)
comps = [0] * s.n_u + [1] * (s.n_vel - s.n_u)
D = sdc.ground_dof(sdc.submatrix(s.matrix, s.n_vel + s.n_pff, s.n_total(), s.n_vel + s.n_pff, s.n_total()))
for name, mat, opts in (("V", V, sdc.AmgOptions(components=comps, max_levels=cfg.v_max_levels)),
                        ("D", D, sdc.AmgOptions(max_levels=cfg.d_max_levels))):
    base = sdc.AmgPreconditioner(mat, opts, ctx=ctx)
    rows = [r for r, _ in base.hierarchy()]
    del base
    variants = [("default", {}), ("no-wave", {"SDG_GS_KNOB_ROWS": str(rows[0]), "SDG_GS_WAVE": "0"}),
                ("lattice", {"SDG_GS_KNOB_ROWS": str(rows[1]), "SDG_GS_LATTICE": "1"})]
    for vname, env in variants:
        for k in ("SDG_GS_KNOB_ROWS", "SDG_GS_WAVE", "SDG_GS_LATTICE"):
            os.environ.pop(k, None)
        os.environ.update(env)
        amg = sdc.AmgPreconditioner(mat, opts, ctx=ctx)
        r = torch.randn(mat.n_rows, dtype=torch.float64, device="cuda")
        z = torch.zeros_like(r)
        def run(k):
            for _ in range(k):
                L.sdg_precond_apply_device(amg.h, C.c_void_p(r.data_ptr()), C.c_void_p(z.data_ptr()))
        run(5)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run(n_app)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / n_app
        print(f"{cfg.name} {name} n={mat.n_rows} {vname:10s} features={sorted(amg.features())} "
              f"{dt * 1e6:.1f} us/apply", flush=True)
        del amg
