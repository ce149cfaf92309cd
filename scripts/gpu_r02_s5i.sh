# session 5: full GPU suite and the other configs with the reworked wavefront kernels
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5i; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest_gpu.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err; echo "c2 rc=$?"
timeout 600 python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc=$?"
timeout 600 python bench.py --config c5s --steps 1 --warmup 0 --coupling-iterations 200 > $O/bench_c5s.json 2> $O/bench_c5s.err; echo "c5s rc=$?"
for f in bench_c2 bench_c4 bench_c5s; do echo "$f: $(tail -1 $O/$f.json | head -c 300)"; done
