# session 5: wavefront start-up experiments (dry passes), chain micro-benchmarks
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5b; mkdir -p $O
./scripts/mb_lat > $O/mb_lat.log 2>&1; head -12 $O/mb_lat.log
./scripts/mb_wavestep > $O/mb_wavestep.log 2>&1; cat $O/mb_wavestep.log
for d in 0 1; do
SDG_WAVE_DRY=$d timeout 300 python scripts/wave_timeline.py c3 V > $O/wave_tl_V_dry$d.log 2>&1; tail -18 $O/wave_tl_V_dry$d.log | cut -c1-250
SDG_WAVE_DRY=$d timeout 300 python scripts/wave_timeline.py c3 D > $O/wave_tl_D_dry$d.log 2>&1; tail -3 $O/wave_tl_D_dry$d.log
SDG_WAVE_DRY=$d timeout 300 python scripts/time_apply.py c3 200 2>&1 | grep -E "us/apply" | sed "s/^/dry=$d /"
done
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "wave or smoother or early" > $O/pytest_wave.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_wave.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
python -c "
import json; d=json.load(open('$O/bench_c3.json')); print('c3', d['ms_per_step'], d['details']['iterations'][:2], {k:(v['launches'],round(v['ms'],1)) for k,v in d['kernel_profile'].items()})"
