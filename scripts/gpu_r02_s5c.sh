# session 5: wavefront with records loaded one step pair ahead
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5c; mkdir -p $O
timeout 300 python scripts/wave_timeline.py c3 V > $O/wave_tl_V.log 2>&1; tail -18 $O/wave_tl_V.log | cut -c1-250
timeout 300 python scripts/wave_timeline.py c3 D > $O/wave_tl_D.log 2>&1; tail -3 $O/wave_tl_D.log
timeout 300 python scripts/time_apply.py c3 200 2>&1 | grep -E "us/apply"
timeout 300 python scripts/time_wave.py c3 2>&1 | tail -8
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "wave or smoother or early or ilu0" > $O/pytest_wave.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_wave.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
python -c "
import json; d=json.load(open('$O/bench_c3.json')); print('c3', d['ms_per_step'], d['details']['iterations'][:2], {k:(v['launches'],round(v['ms'],1)) for k,v in d['kernel_profile'].items()})"
