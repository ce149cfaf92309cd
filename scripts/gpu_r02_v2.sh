# nested-dissection coarse solve: kernel tests, c3 / c2 bench, c4 run
cd $GRAFT_REPO_ROOT
O=gpurun_out/v2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "lu_ or nd_ or amg or td_bgs or block_kinds" > $O/pytest_lu.log 2>&1; echo "pytest lu rc=$?"
tail -5 $O/pytest_lu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
SDG_COARSE=dense timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c3_dense.json 2> $O/bench_c3_dense.err; echo "c3 dense rc=$?"
timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err; echo "c2 rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 $O/pytest_gpu.log
timeout 900 python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc=$?"
python - <<'P'
import json
for f in ("bench_c3","bench_c3_dense","bench_c2","bench_c4"):
    try:
        d=json.load(open(f"gpurun_out/v2/{f}.json"))
        print(f, d["ms_per_step"], d["value"], (d.get("details") or d.get("config")).get("iterations", (d.get("details") or d.get("config")).get("iterations_per_time_step")), (d.get("details") or {}).get("setup_s"))
        print("   coarse", d.get("kernel_profile",{}).get("coarse"))
    except Exception as e:
        print(f, "ERR", e)
P
