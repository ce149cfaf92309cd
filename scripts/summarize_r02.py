"""Dev helper: copy one validation run (gpurun_out/<dir>, scripts/gpu_r02_v*.sh) into
profiles/r02/ and refresh profiles/ncu_traffic.json (DRAM bytes per launch of the
kernel families bench.py reports a roofline for, from the ncu passes of that run).

    python scripts/summarize_r02.py gpurun_out/v1
"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.abspath(sys.argv[1])
DST = os.path.join(ROOT, "profiles", "r02")
os.makedirs(DST, exist_ok=True)


def rows(path):
    with open(path) as f:
        return list(csv.DictReader(l for l in f if not l.startswith("==")))


def short(name):
    n = name.split("(")[0].replace("void ", "").strip()
    return n.split("::")[-1]


def details(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    out = []
    for r in csv.DictReader(txt.splitlines()):
        if r.get("Metric Name"):
            out.append(r)
    launches = collections.OrderedDict()
    for r in out:
        l = launches.setdefault(r["ID"], {"kernel": short(r["Kernel Name"]), "grid": r.get("Grid Size"),
                                          "block": r.get("Block Size"), "sections": {}})
        l["sections"].setdefault(r["Section Name"], {})[r["Metric Name"]] = (r["Metric Value"] + " " + r["Metric Unit"]).strip()
    return list(launches.values())


for f in ("bench_c3.json", "bench_c2.json", "bench_c4.json", "pytest_gpu.log", "smoke.log", "apply_dram_c3.csv"):
    if os.path.exists(os.path.join(SRC, f)):
        shutil.copy(os.path.join(SRC, f), os.path.join(DST, f))

# launch list of `bench.py --steps 1 --warmup 3` (the timed solve): per-kernel summary + the raw list
ll = os.path.join(SRC, "launches_c3.csv")
if os.path.exists(ll):
    shutil.copy(ll, os.path.join(DST, "launches_c3.csv"))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows(ll):
        a = agg[short(r["Kernel Name"])]
        a[0] += 1
        a[1] += float(r["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    with open(os.path.join(DST, "launches_c3_summary.csv"), "w") as f:
        f.write("kernel,launches,total_ms,mean_us,share_of_kernel_time\n")
        for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"\"{k}\",{c},{t / 1e6:.3f},{t / c / 1e3:.2f},{t / tot:.4f}\n")

# DRAM bytes per launch of one td_bgs apply (ncu, caches cold per launch)
traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
try:
    traffic = json.load(open(traffic_path))
except Exception:
    traffic = {}
ad = os.path.join(SRC, "apply_dram_c3.csv")
if os.path.exists(ad):
    per = collections.OrderedDict()
    for r in rows(ad):
        d = per.setdefault(r["ID"], {"k": short(r["Kernel Name"])})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    fam = {"gs_wave": "k_gs_wave", "gs": "k_gs_walk", "coarse": ("k_dense_gemv", "k_nd_"), "iface": "k_colmajor_gemv_sub",
           "gsprep": "k_gs_prep", "restrict": "k_restrict_warp"}
    for name, pat in fam.items():
        pats = pat if isinstance(pat, tuple) else (pat,)
        ls = [d for d in per.values() if any(d["k"].startswith(p) for p in pats)]
        if not ls:
            continue
        b = sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in ls) / len(ls)
        traffic[name] = {"config": "c3", "kernel": f"{'/'.join(sorted(set(d['k'] for d in ls)))}: mean over the {len(ls)} "
                         f"launches of one td_bgs apply, c3",
                         "dram_bytes_per_launch": b,
                         "source": "profiles/r02/apply_dram_c3.csv (ncu --profile-from-start off --metrics gpu__time_duration.sum,"
                                   "dram__bytes_read.sum,dram__bytes_write.sum over one apply; caches cold per launch)"}
for name, rep in (("ncu_gs_wave_c3.json", "gs_wave_c3.ncu-rep"), ("ncu_gs_walk_c3.json", "gs_walk_c3.ncu-rep"),
                  ("ncu_dense_gemv_c3.json", "dense_gemv_c3.ncu-rep"), ("ncu_nd_c3.json", "nd_c3.ncu-rep")):
    p = os.path.join(SRC, rep)
    if os.path.exists(p):
        with open(os.path.join(DST, name), "w") as f:
            json.dump({"report": rep, "command": "ncu --profile-from-start off --set full --clock-control none "
                       "--import-source on -k regex:<kernel> -c 2 python scripts/prof_apply.py c3",
                       "launches": details(p)}, f, indent=1)
with open(traffic_path, "w") as f:
    json.dump(traffic, f, indent=2)
print(json.dumps(traffic, indent=1)[:2000])
