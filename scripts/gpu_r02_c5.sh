# config 5 at its size (2000^2 per subdomain): the first two coupling iterations
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02c5
timeout 900 python -m pytest tests/test_gpu_solvers.py -q -k "ilu0" > gpurun_out/r02c5/pytest_ilu0.log 2>&1
echo "ilu0 rc=$?"
timeout 1800 python bench.py --config c5 --steps 1 --warmup 0 --coupling-iterations 2 > gpurun_out/r02c5/bench_c5_k2.json 2> gpurun_out/r02c5/bench_c5_k2.err
echo "c5 rc=$?"
SDG_GS_LATTICE=1 timeout 1800 python bench.py --config c5 --steps 1 --warmup 0 --coupling-iterations 2 > gpurun_out/r02c5/bench_c5_k2_lattice.json 2> gpurun_out/r02c5/bench_c5_k2_lattice.err
echo "c5 lattice rc=$?"
tail -2 gpurun_out/r02c5/pytest_ilu0.log
