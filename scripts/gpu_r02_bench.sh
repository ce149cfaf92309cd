cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02b
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py -x -q > gpurun_out/r02b/pytest.log 2>&1
echo "pytest rc=$?"
timeout 400 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02b/bench_c3.json 2> gpurun_out/r02b/bench_c3.err
echo "c3 rc=$?"
timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02b/bench_c2.json 2> gpurun_out/r02b/bench_c2.err
echo "c2 rc=$?"
tail -2 gpurun_out/r02b/pytest.log
