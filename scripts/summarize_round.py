"""Dev helper: copy a gpu_round.sh run (gpurun_out/r) into profiles/<round>/ and
refresh profiles/ncu_traffic.json (DRAM bytes per launch of the kernel
families the bench reports a roofline for)."""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "r")
DST = os.path.join(ROOT, "profiles", sys.argv[1] if len(sys.argv) > 1 else "r01")


def rows(path):
    with open(path) as f:
        return list(csv.DictReader(l for l in f if not l.startswith("==")))


def per_launch(path):
    out = {}
    for r in rows(path):
        k = r["ID"]
        d = out.setdefault(k, {"kernel": r["Kernel Name"], "stream": r.get("Stream", "")})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return list(out.values())


def details(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    sec = {}
    for r in csv.DictReader(txt.splitlines()):
        if r.get("Metric Name"):
            sec.setdefault(r["Section Name"], {})[r["Metric Name"]] = (r["Metric Value"] + " " + r["Metric Unit"]).strip()
    return sec


os.makedirs(DST, exist_ok=True)
for f in ("bench.json", "bench_ref.json", "bench_c3.json", "bench_c4.json", "pytest_gpu.log", "smoke.log"):
    if os.path.exists(os.path.join(SRC, f)):
        shutil.copy(os.path.join(SRC, f), os.path.join(DST, f))
shutil.copy(os.path.join(SRC, "launches.csv"), os.path.join(DST, "launches_c2.csv"))
shutil.copy(os.path.join(SRC, "apply_dram.csv"), os.path.join(DST, "apply_dram_c2.csv"))
traffic = {}
walks = [l for l in per_launch(os.path.join(SRC, "apply_dram.csv")) if "k_gs_walk" in l["kernel"]]
if walks:
    b = sum(l["dram__bytes_read.sum"] + l["dram__bytes_write.sum"] for l in walks) / len(walks)
    traffic["gs"] = {"kernel": f"k_gs_walk, mean over the {len(walks)} walk launches of one td_bgs apply, c2",
                     "dram_bytes_per_launch": b,
                     "source": "profiles/r01/apply_dram_c2.csv (ncu --profile-from-start off --metrics "
                               "dram__bytes_read.sum,dram__bytes_write.sum over one apply; caches cold per launch)"}
for name, rep, fam in (("ncu_gs_walk_v0.json", "gs_walk_v0.ncu-rep", None), ("ncu_spmv_c3.json", "spmv_c3.ncu-rep", "spmv"),
                       ("ncu_gemv_c3.json", "gemv_c3.ncu-rep", "gemv")):
    p = os.path.join(SRC, rep)
    if not os.path.exists(p):
        continue
    sec = details(p)
    with open(os.path.join(DST, name), "w") as f:
        json.dump({"report": rep, "sections": sec}, f, indent=1)
    if fam:
        raw = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv", "--metrics",
                              "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
        rr = list(csv.reader(raw.splitlines()))
        hdr, units, vals = rr[0], rr[1], rr[2]
        tot = 0.0
        for h, u, v in zip(hdr, units, vals):
            if h in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                tot += float(v.replace(",", "")) * scale
        what = {"spmv": "k_spmv_sell (operator SpMV, SELL-32), c3, one launch",
                "gemv": "k_colmajor_gemv_sub (td_bgs interface GEMV, K 250,000 x 500), c3, one launch"}[fam]
        traffic[fam] = {"kernel": what, "dram_bytes_per_launch": tot,
                        "source": f"profiles/r01/{name} (ncu --set full)"}
with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
    json.dump(traffic, f, indent=2)
print(json.dumps(traffic, indent=1))
