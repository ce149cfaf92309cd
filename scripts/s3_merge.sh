# level-merging experiment: decisions, bench per forced k, GPU tests
mkdir -p gpurun_out/m
SDG_DEBUG=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/m/auto.json 2> gpurun_out/m/auto.err
for k in 1 2 3 4 6; do
  SDG_GS_MERGE=$k timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/m/k$k.json 2> gpurun_out/m/k$k.err
done
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_solvers.py::test_c3_full_size_matches_reference_fingerprint > gpurun_out/m/pytest.log 2>&1; echo "exit $?" >> gpurun_out/m/pytest.log
