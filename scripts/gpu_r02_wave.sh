# round 2: first run of the multi-SM wavefront smoother + GMRES graphs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02w
export SDG_DEBUG=0
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/r02w/pytest_kernels.log 2>&1
echo "kernels rc=$?"
timeout 600 python -m pytest tests/test_gpu_solvers.py -x -q > gpurun_out/r02w/pytest_solvers.log 2>&1
echo "solvers rc=$?"
timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02w/bench_c3.json 2> gpurun_out/r02w/bench_c3.err
echo "c3 rc=$?"
timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02w/bench_c2.json 2> gpurun_out/r02w/bench_c2.err
echo "c2 rc=$?"
tail -3 gpurun_out/r02w/*.log
