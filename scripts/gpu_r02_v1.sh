# round 2 validation at HEAD: GPU tests, smoke, c3 bench, ncu launch list of the bench command,
# per-apply DRAM bytes, full captures of the dominant kernels (wavefront, coarse walk, coarse GEMV)
cd $GRAFT_REPO_ROOT
O=gpurun_out/v1; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
# launch list of the bench command (the timed solve only: cudaProfilerStart/Stop around it)
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/plain_small.log 2>&1 && \
SDG_PROFILER_RANGE=1 timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $O/launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
echo "launch list rc=$?"
SDG_PROFILER_RANGE=1 timeout 900 ncu --profile-from-start off --clock-control none --csv --log-file $O/apply_dram_c3.csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum python scripts/prof_apply.py c3 > $O/ncu_apply.log 2>&1
echo "apply dram rc=$?"
SDG_PROFILER_RANGE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:k_gs_wave -c 2 -f -o $O/gs_wave_c3 python scripts/prof_apply.py c3 > $O/ncu_wave.log 2>&1
SDG_PROFILER_RANGE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:k_gs_walk -c 2 -f -o $O/gs_walk_c3 python scripts/prof_apply.py c3 > $O/ncu_walk.log 2>&1
SDG_PROFILER_RANGE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:k_dense_gemv -c 2 -f -o $O/dense_gemv_c3 python scripts/prof_apply.py c3 > $O/ncu_gemv.log 2>&1
echo "ncu full done"
tail -3 $O/pytest_gpu.log; cat $O/smoke.log | tail -1; head -c 600 $O/bench_c3.json
