# multi-warp wavefront / lattice CTAs: bitwise tests, then c3 apply and solve timings per variant
cd $GRAFT_REPO_ROOT
O=gpurun_out/v4; mkdir -p $O
for W in 1 2 4; do
  SDG_WAVE_W=$W timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "wave_smoother" > $O/pytest_wave_w$W.log 2>&1; echo "wave W=$W rc=$? $(tail -1 $O/pytest_wave_w$W.log)"
done
for W in 1 2 3 4; do
  SDG_LAT_W=$W timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "lattice" > $O/pytest_lat_w$W.log 2>&1; echo "lattice W=$W rc=$? $(tail -1 $O/pytest_lat_w$W.log)"
done
echo "--- applies (us/apply), c3"
SDG_WAVE_W=1 SDG_GS_LATTICE=0 timeout 300 python scripts/time_apply.py c3 100 2>&1 | tail -1 | sed 's/^/waveW1 lat0: /'
SDG_GS_LATTICE=0 timeout 300 python scripts/time_apply.py c3 100 2>&1 | tail -1 | sed 's/^/waveWdef lat0: /'
for W in 1 2 3 4; do
  SDG_LAT_W=$W SDG_GS_LATTICE=1 timeout 300 python scripts/time_apply.py c3 100 2>&1 | tail -1 | sed "s/^/waveWdef lat1 W$W: /"
done
SDG_DEBUG=1 timeout 300 python scripts/time_apply.py c3 100 2>&1 | grep -E "label block|us/apply|lattice\]|gs wave" | sed 's/^/auto: /'
SDG_LAT_W=3 SDG_DEBUG=1 timeout 300 python scripts/time_apply.py c3 100 2>&1 | grep -E "label block|us/apply" | sed 's/^/auto W3: /'
SDG_LAT_W=4 SDG_DEBUG=1 timeout 300 python scripts/time_apply.py c3 100 2>&1 | grep -E "label block|us/apply" | sed 's/^/auto W4: /'
echo "--- solves"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c3_auto.json 2> $O/bench_c3_auto.err; echo "c3 auto rc=$?"
SDG_GS_LATTICE=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c3_lat0.json 2> $O/bench_c3_lat0.err; echo "c3 lat0 rc=$?"
SDG_GS_LATTICE=0 SDG_WAVE_W=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c3_old.json 2> $O/bench_c3_old.err; echo "c3 old rc=$?"
python - <<'P'
import json
for f in ("bench_c3_auto","bench_c3_lat0","bench_c3_old"):
    try:
        d=json.load(open(f"gpurun_out/v4/{f}.json"))
        kp=d["kernel_profile"]
        print(f, round(d["ms_per_step"],1), d["details"]["iterations"][:2], {k:(v["launches"],round(v["ms"],1)) for k,v in kp.items() if k in("gs","gs_wave","gs_lattice","coarse")}, d["details"].get("fast_paths"))
    except Exception as e:
        print(f,"ERR",e)
P
