# session 5: multi-dot without per-group barriers (test + c3), then the complete launch list at HEAD
cd $GRAFT_REPO_ROOT
O=gpurun_out/final; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_solvers.py -m gpu -q -x > $O/pytest_solvers.log 2>&1; echo "solver tests rc=$?"; tail -2 $O/pytest_solvers.log
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_c3_md.json 2> $O/bench_c3_md.err; echo "c3 rc=$?"
python -c "
import json; d=json.loads(open('$O/bench_c3_md.json').read().strip().splitlines()[-1]); print('c3', d['ms_per_step'], d['e2e']['ms_per_step'], d['details']['iterations'][:2], d['kernel_profile']['ortho'])"
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/plain_small.log 2>&1 && \
SDG_PROFILER_RANGE=1 timeout 2400 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $O/launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
echo "launch list rc=$?"; grep -c gpu__time_duration $O/launches_c3.csv
