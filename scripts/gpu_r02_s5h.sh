cd $GRAFT_REPO_ROOT
O=gpurun_out/s5h; mkdir -p $O
for sp in 0 1; do
echo "SDG_WAVE_SPLIT=$sp"; SDG_WAVE_SPLIT=$sp timeout 120 python scripts/time_wave.py c3 2>&1 | grep "V.*default" || { echo "time_wave failed/hung"; }
done
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "wave or smoother or early or ilu0" > $O/pytest_wave.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_wave.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
python -c "
import json; d=json.load(open('$O/bench_c3.json')); print('c3', d['ms_per_step'], d['details']['iterations'][:2], {k:(v['launches'],round(v['ms'],1)) for k,v in d['kernel_profile'].items()})"
SDG_WAVE_W=1 timeout 120 python scripts/wave_timeline.py c3 V 2>&1 | tail -17 | cut -c1-90
