"""Dev aid: per-band timeline of the last wavefront launch (SDG_WAVE_TL=1):
one AMG apply of the velocity (MAC) or porous (5-point) block of a config,
then {start, first block, end, waiting} per band relative to the first start.
python scripts/wave_timeline.py c3 V|D"""
import ctypes as C, os, sys
os.environ["SDG_WAVE_TL"] = "1"
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2108_13229_b200 import scenarios, sdc
cfg = scenarios.CONFIGS[sys.argv[1]]
which = sys.argv[2] if len(sys.argv) > 2 else "V"
s = scenarios.build_system(cfg)
if which == "V":
    mat = sdc.submatrix(s.matrix, 0, s.n_vel, 0, s.n_vel)
    amg = sdc.AmgPreconditioner(mat, sdc.AmgOptions(components=[0] * s.n_u + [1] * (s.n_vel - s.n_u),
                                                    max_levels=cfg.v_max_levels))
else:
    mat = sdc.ground_dof(sdc.submatrix(s.matrix, s.n_vel + s.n_pff, s.n_total(), s.n_vel + s.n_pff, s.n_total()))
    amg = sdc.AmgPreconditioner(mat, sdc.AmgOptions(max_levels=cfg.d_max_levels))
r = np.random.default_rng(1).standard_normal(mat.n_rows)
for _ in range(3):
    amg.apply(r)
L = sdc.lib()
buf = (C.c_ulonglong * 8192)()
nb = L.sdg_debug_wave_timeline(buf, 1024)
t = np.array(buf[: 8 * nb], dtype=np.float64).reshape(nb, 8)
t0 = t[:, 0].min()
print(f"{cfg.name} {which}: {nb} bands, last wave launch (the post-smoother), ns from the first band start")
for b in range(nb):
    print(f"band {b:3d}: start {t[b,0]-t0:9.0f} first {t[b,1]-t0:9.0f} end {t[b,2]-t0:9.0f} "
          f"run {t[b,2]-t[b,1]:9.0f} wait cyc {t[b,3]:9.0f} tma-wait cyc {t[b,4]:9.0f} compute cyc {t[b,5]:9.0f} "
          f"first->blk4 {t[b,6]-t[b,1]:7.0f} blk4->blk12 {t[b,7]-t[b,6]:7.0f}")
print(f"total {t[:,2].max()-t0:.0f} ns")

if os.environ.get("SDG_WAVE_TL_BLOCKS"):
    bb = (C.c_ulonglong * (128 * 1024))()
    nb2 = L.sdg_debug_wave_blocks(bb, 1024)
    B = np.array(bb[: 128 * nb2], dtype=np.float64).reshape(nb2, 128) - t0
    nq = int((B[0] > -1e17).sum()) if False else int(os.environ["SDG_WAVE_TL_BLOCKS"])
    np.save(os.path.join("gpurun_out", "s5e", f"blocks_{which}_w{os.environ.get('SDG_WAVE_W', 'd')}.npy"), B[:, :nq])
    print("block start times (us), rows = bands, every 4th block; then lag to the band below")
    for b in range(min(nb2, 6)):
        print(f"band {b}: " + " ".join(f"{B[b, q] / 1e3:6.1f}" for q in range(0, nq, 4)))
    for b in range(1, min(nb2, 6)):
        print(f"lag {b}-{b-1}: " + " ".join(f"{(B[b, q] - B[b - 1, q]) / 1e3:6.1f}" for q in range(0, nq, 4)))
