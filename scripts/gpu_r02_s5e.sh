cd $GRAFT_REPO_ROOT
O=gpurun_out/s5e; mkdir -p $O
SDG_WAVE_TL_BLOCKS=34 timeout 300 python scripts/wave_timeline.py c3 D > $O/wave_tl_D_w4.log 2>&1; grep -E "band +(0|1|2|15):|total" $O/wave_tl_D_w4.log | cut -c1-150
SDG_WAVE_TL_BLOCKS=67 SDG_WAVE_W=1 timeout 300 python scripts/wave_timeline.py c3 V > $O/wave_tl_V_w1.log 2>&1;  grep -E "band +(0|1|2|15):|total" $O/wave_tl_V_w1.log | cut -c1-150
SDG_WAVE_TL_BLOCKS=67 SDG_WAVE_W=2 timeout 300 python scripts/wave_timeline.py c3 V > $O/wave_tl_V_w2.log 2>&1;  grep -E "band +(0|1|2|15):|total" $O/wave_tl_V_w2.log | cut -c1-150
timeout 300 python scripts/time_wave.py c3 2>&1 | tail -8
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "wave or smoother or early or ilu0" > $O/pytest_wave.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_wave.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
python -c "
import json; d=json.load(open('$O/bench_c3.json')); print('c3', d['ms_per_step'], d['details']['iterations'][:2], {k:(v['launches'],round(v['ms'],1)) for k,v in d['kernel_profile'].items()})"
