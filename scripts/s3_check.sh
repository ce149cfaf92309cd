mkdir -p gpurun_out/s3
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s3/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/s3/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/s3/smoke.log
timeout 600 python bench.py > gpurun_out/s3/bench.json 2> gpurun_out/s3/bench.err; echo "bench exit $?" >> gpurun_out/s3/bench.err
