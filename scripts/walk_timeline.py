"""Dev helper (library built with -DSDG_WALK_TL): globaltimer timeline of the
walk kernels of a few device-resident td_bgs applies (config argv[1], default c2)."""
import os, sys
import ctypes as C
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2108_13229_b200 import scenarios, sdc
cfg = scenarios.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
s = scenarios.build_system(cfg)
ctx = sdc.default_context()
p = sdc.TdPreconditioner(s, "td_bgs", cfg.v_max_levels, cfg.d_max_levels, ctx=ctx)
r = torch.randn(s.n_total(), dtype=torch.float64, device="cuda")
z = torch.zeros_like(r)
L = sdc.lib()
buf = (C.c_ulonglong * (4 * 4096))()
for _ in range(5):
    L.sdg_precond_apply_device(p.h, C.c_void_p(r.data_ptr()), C.c_void_p(z.data_ptr()))
torch.cuda.synchronize()
L.sdg_debug_walk_timeline(buf, 4096)
for _ in range(3):
    L.sdg_precond_apply_device(p.h, C.c_void_p(r.data_ptr()), C.c_void_p(z.data_ptr()))
torch.cuda.synchronize()
m = L.sdg_debug_walk_timeline(buf, 4096)
a = np.frombuffer(buf, dtype=np.uint64)[: 4 * m].reshape(m, 4).astype(np.int64)
t0 = a[:, 0].min()
for row in sorted(a.tolist(), key=lambda x: x[0]):
    print(f"start {(row[0]-t0)/1e3:8.1f} us  wait-done {(row[1]-t0)/1e3:8.1f}  end {(row[2]-t0)/1e3:8.1f}  "
          f"dur {(row[2]-row[1])/1e3:6.1f}  sm {row[3] & 0xffff:3d}  levels {row[3] >> 16}")
