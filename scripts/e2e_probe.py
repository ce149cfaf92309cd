"""Dev probe: wall time of device-pointer vs host-pointer solves of a config,
alternating (python scripts/e2e_probe.py c3)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2108_13229_b200 import scenarios, sdc
cfg = scenarios.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
s = scenarios.build_system(cfg)
ctx = sdc.default_context()
p = sdc.TdPreconditioner(s, "td_bgs", cfg.v_max_levels, cfg.d_max_levels, ctx=ctx)
tol = 1e-8 * float(np.linalg.norm(s.rhs))
ctrl = sdc.RestartController.fixed(50)
b_dev = torch.from_numpy(s.rhs).cuda()
x_dev = torch.zeros_like(b_dev)
b_pin = torch.from_numpy(s.rhs.copy()).pin_memory().numpy()
for k in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = sdc.pd_gmres_device(s.matrix, p, b_dev.data_ptr(), x_dev.data_ptr(), tol, 4000, ctrl, ctx=ctx)
    t1 = time.perf_counter()
    res = sdc.pd_gmres(s.matrix, p, b_pin, tol, 4000, ctrl)
    t2 = time.perf_counter()
    print(f"device {1e3*(t1-t0):.1f} ms ({rep.iterations} it, device_ms {rep.device_ms:.1f})  "
          f"host {1e3*(t2-t1):.1f} ms ({res.report.iterations} it, device_ms {res.report.device_ms:.1f})", flush=True)
