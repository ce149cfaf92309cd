# round 2, session 5: final measurement at HEAD (reworked wavefront kernels): GPU tests, smoke,
# the driver's c3 bench command (with the cpu_baseline leg), ncu launch list of the bench command,
# per-apply DRAM bytes, full captures of the dominant kernels, then the other configs' bench lines
cd $GRAFT_REPO_ROOT
O=gpurun_out/final; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/plain_small.log 2>&1 && \
SDG_PROFILER_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $O/launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
echo "launch list rc=$?"
SDG_PROFILER_RANGE=1 timeout 600 ncu --profile-from-start off --clock-control none --csv --log-file $O/apply_dram_c3.csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum python scripts/prof_apply.py c3 > $O/ncu_apply.log 2>&1
echo "apply dram rc=$?"
SDG_PROFILER_RANGE=1 timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:k_gs_wave_mac -c 2 -f -o $O/gs_wave_c3 python scripts/prof_apply.py c3 > $O/ncu_wave.log 2>&1
SDG_PROFILER_RANGE=1 timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:k_gs_walk -c 2 -f -o $O/gs_walk_c3 python scripts/prof_apply.py c3 > $O/ncu_walk.log 2>&1
SDG_PROFILER_RANGE=1 timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:k_nd_ -c 16 -f -o $O/nd_c3 python scripts/prof_apply.py c3 > $O/ncu_nd.log 2>&1
echo "ncu full done"
timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err; echo "c2 rc=$?"
timeout 600 python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc=$?"
timeout 600 python bench.py --config c5s --steps 1 --warmup 0 --coupling-iterations 200 > $O/bench_c5s.json 2> $O/bench_c5s.err; echo "c5s rc=$?"
timeout 400 python bench.py --sharded --config c3 --steps 5 --warmup 2 > $O/bench_sharded_c3_n1.json 2> $O/bench_sharded_c3_n1.err; echo "sharded rc=$?"
for f in bench_c3 bench_c2 bench_c4 bench_c5s bench_sharded_c3_n1; do echo "$f: $(tail -1 $O/$f.json | head -c 260)"; done
timeout 1200 python bench.py --config c5 --steps 1 --warmup 0 --coupling-iterations 2 > $O/bench_c5_first2.json 2> $O/bench_c5_first2.err; echo "c5 rc=$?"
echo "c5: $(tail -1 $O/bench_c5_first2.json | head -c 400)"; grep "\[dn\]" $O/bench_c5_first2.err | tail -4
SDG_DEBUG=1 timeout 300 python scripts/time_apply.py c3 100 2>&1 | grep -E "label block|us/apply|gs wave" | sed 's/^/c3 plan: /'
# the driver's own command, cpu_baseline leg included (its reference setup runs ~11 min beside the GPU work)
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "driver-style bench rc=$?"; tail -1 $O/bench.json | head -c 600
