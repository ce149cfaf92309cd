# the driver's own bench command at the final build (cpu_baseline leg included)
cd $GRAFT_REPO_ROOT
O=gpurun_out/final; mkdir -p $O
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "driver-style bench rc=$?"; tail -1 $O/bench.json | head -c 400
