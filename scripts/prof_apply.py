"""Dev helper: c2 system, td_bgs preconditioner, timed applies + per-family profile.

With SDG_PROFILER_RANGE=1 the last apply is wrapped in cudaProfilerStart/Stop,
so `ncu --profile-from-start off` captures exactly one preconditioner apply."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2108_13229_b200 import scenarios, sdc
cfg = scenarios.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
s = scenarios.build_system(cfg)
ctx = sdc.default_context()
p = sdc.TdPreconditioner(s, "td_bgs", cfg.v_max_levels, cfg.d_max_levels, ctx=ctx)
r = np.random.default_rng(0).standard_normal(s.n_total())
for _ in range(3):
    p.apply(r)
ctx.set_profiling(True)
for _ in range(5):
    p.apply(r)
prof = ctx.profile()
ctx.set_profiling(False)
for k, v in prof.items():
    print(f"{k:10s} launches/apply={v['launches']/5:6.1f} ms/apply={v['ms']/5:8.3f} GB/s={v['bytes']/v['ms']/1e6:8.1f}")
print("hier", p.hierarchy(0), p.hierarchy(1))
if os.environ.get("SDG_PROFILER_RANGE"):
    import torch
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    p.apply(r)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
