"""Dev probe: warm-started transient steps of a config on the GPU (prints per step)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2108_13229_b200 import drivers, scenarios
cfg = scenarios.CONFIGS[sys.argv[1]]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.steps
if len(sys.argv) > 3:
    import dataclasses
    cfg = dataclasses.replace(cfg, solver=sys.argv[3])
drv = drivers.TransientDriver(cfg, warm_start=True)
for k in range(1, steps + 1):
    try:
        st = drv.advance(k * cfg.dt)
        print(k, st.iterations, st.converged, round(st.solve_seconds, 2), flush=True)
    except Exception as e:
        print(k, "EXC", e, flush=True)
        break
