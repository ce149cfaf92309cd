# round 2 measurement session: GPU tests, bench lines of every config, reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02r
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02r/pytest_gpu.log 2>&1
echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02r/smoke.log 2>&1
echo "smoke rc=$?"
timeout 600 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02r/bench_c3.json 2> gpurun_out/r02r/bench_c3.err
echo "c3 rc=$?"
timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02r/bench_c2.json 2> gpurun_out/r02r/bench_c2.err
echo "c2 rc=$?"
timeout 900 python bench.py --config c4 --steps 1 --warmup 0 > gpurun_out/r02r/bench_c4.json 2> gpurun_out/r02r/bench_c4.err
echo "c4 rc=$?"
timeout 900 python bench.py --config c5s --steps 1 --warmup 0 --coupling-iterations 200 > gpurun_out/r02r/bench_c5s.json 2> gpurun_out/r02r/bench_c5s.err
echo "c5s rc=$?"
timeout 600 python bench.py --sharded --config c3 --steps 5 --warmup 2 > gpurun_out/r02r/bench_sharded_c3_n1.json 2> gpurun_out/r02r/bench_sharded_c3_n1.err
echo "sharded rc=$?"
tail -3 gpurun_out/r02r/pytest_gpu.log
