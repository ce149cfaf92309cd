"""Dev helper: wall time of N device-resident td_bgs applies on c2 (env knobs
such as SDG_TD_OVERLAP / SDG_GS_MERGE select the variant)."""
import os, sys, time
import ctypes as C
sys.path.insert(0, os.getcwd())
import torch
from paper_2108_13229_b200 import scenarios, sdc
cfg = scenarios.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
n_app = int(sys.argv[2]) if len(sys.argv) > 2 else 200
s = scenarios.build_system(cfg)
ctx = sdc.default_context()
p = sdc.TdPreconditioner(s, "td_bgs", cfg.v_max_levels, cfg.d_max_levels, ctx=ctx)
r = torch.randn(s.n_total(), dtype=torch.float64, device="cuda")
z = torch.zeros_like(r)
L = sdc.lib()
def run(k):
    for _ in range(k):
        L.sdg_precond_apply_device(p.h, C.c_void_p(r.data_ptr()), C.c_void_p(z.data_ptr()))
run(10)
torch.cuda.synchronize()
best = 1e9
for rep in range(3):
    t0 = time.perf_counter()
    run(n_app)
    t_enq = (time.perf_counter() - t0) / n_app
    torch.cuda.synchronize()
    best = min(best, (time.perf_counter() - t0) / n_app)
enq = []
for _ in range(50):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(1)
    enq.append(time.perf_counter() - t0)
enq.sort()
print(f"single-apply host enqueue median {enq[25] * 1e6:.1f} us")
print(f"{os.environ.get('SDG_TD_OVERLAP', '-')} {os.environ.get('SDG_GS_MERGE', '-')} us/apply {best * 1e6:.1f} "
      f"(host enqueue {t_enq * 1e6:.1f} us/apply)  |z|={z.norm().item():.12e}")
