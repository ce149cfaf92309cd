"""Dev/checker aid: per-step BiCGSTAB iteration counts (and breakdown restarts) of the c4s
transient on the GPU under the variants named on the command line (env knobs are set by
the caller); prints one JSON line.  python scripts/c4s_variants.py <label> [seed]"""
import json, os, sys
sys.path.insert(0, os.getcwd())
from paper_2108_13229_b200 import drivers, scenarios
label = sys.argv[1]
seed = int(sys.argv[2]) if len(sys.argv) > 2 else None
cfg = scenarios.CONFIGS["c4s"]
drv = drivers.TransientDriver(cfg, warm_start=True, rhs_perturbation_seed=seed)
hist = drv.run()
print(json.dumps({"variant": label, "seed": seed, "iterations": [h.iterations for h in hist],
                  "restarts": [h.breakdown_restarts for h in hist], "total": sum(h.iterations for h in hist)}))
