"""Dev helper: build a config's preconditioner and time applies per kernel family
(cudaProfilerStart/Stop around one apply with SDG_PROFILER_RANGE=1)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2108_13229_b200 import scenarios, sdc
cfg = scenarios.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
s = scenarios.build_system(cfg)
ctx = sdc.default_context()
t0 = time.perf_counter()
p = sdc.TdPreconditioner(s, "td_bgs", cfg.v_max_levels, cfg.d_max_levels, ctx=ctx)
print("setup s", time.perf_counter() - t0)
r = np.random.default_rng(0).standard_normal(s.n_total())
p.apply(r)
ctx.set_profiling(True)
for _ in range(2):
    p.apply(r)
prof = ctx.profile()
ctx.set_profiling(False)
for k, v in prof.items():
    print(f"{k:10s} launches/apply={v['launches']/2:6.1f} ms/apply={v['ms']/2:8.3f} GB/s={v['bytes']/v['ms']/1e6:8.1f}")
if os.environ.get("SDG_PROFILER_RANGE"):
    import torch
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    p.apply(r)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
