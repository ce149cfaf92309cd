# session 5 baseline at HEAD: plan timings, wave timeline, c3 bench with profile, GPU suite
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5a; mkdir -p $O
SDG_DEBUG=1 timeout 300 python scripts/time_apply.py c3 100 > $O/time_apply_c3.log 2>&1
grep -E "label block|us/apply|gs wave|lattice" $O/time_apply_c3.log | head -30
timeout 300 python scripts/wave_timeline.py c3 V > $O/wave_tl_V.log 2>&1; tail -20 $O/wave_tl_V.log
timeout 300 python scripts/wave_timeline.py c3 D > $O/wave_tl_D.log 2>&1; tail -6 $O/wave_tl_D.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
python -c "
import json; d=json.load(open('$O/bench_c3.json')); print('c3', d['ms_per_step'], d['details']['iterations'][:2], {k:(v['launches'],round(v['ms'],1)) for k,v in d['kernel_profile'].items()})"
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest_gpu.log
