mkdir -p gpurun_out/q
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/q/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/q/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/q/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/q/smoke.log
timeout 600 python bench.py > gpurun_out/q/bench.json 2> gpurun_out/q/bench.err; echo "bench exit $?" >> gpurun_out/q/bench.err
tail -3 gpurun_out/q/pytest_gpu.log; cat gpurun_out/q/bench.json | head -c 600
