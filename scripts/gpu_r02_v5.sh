# full GPU suite at HEAD, planner diagnostics at c3, strip-path A/B (coarse dense vs nd)
cd $GRAFT_REPO_ROOT
O=gpurun_out/v5; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest_gpu.log
SDG_DEBUG=1 timeout 300 python scripts/one_apply.py c3 V 1 2>&1 | grep -E "gs walk|gs plan|gs merge|lattice" | head -30
echo "--- sharded A/B"
timeout 600 python bench.py --sharded --config c3 --steps 5 --warmup 2 --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('nd', d['ms_per_step'], d['gpu_launches'])"
SDG_COARSE=dense timeout 600 python bench.py --sharded --config c3 --steps 5 --warmup 2 --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('dense', d['ms_per_step'], d['gpu_launches'])"
timeout 600 python bench.py --sharded --config c3 --steps 5 --warmup 2 --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('nd again', d['ms_per_step'], d['gpu_launches'])"
