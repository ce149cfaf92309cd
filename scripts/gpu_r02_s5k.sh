# session 5: device matrix assembly test, complete ncu launch list of the bench command
cd $GRAFT_REPO_ROOT
O=gpurun_out/final; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_transient.py -m gpu -q -x -k "assembly" > $O/pytest_assembly.log 2>&1; echo "assembly tests rc=$?"; tail -3 $O/pytest_assembly.log
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/plain_small.log 2>&1 && \
SDG_PROFILER_RANGE=1 timeout 2400 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $O/launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
echo "launch list rc=$?"; grep -c gpu__time_duration $O/launches_c3.csv
