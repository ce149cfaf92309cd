mkdir -p gpurun_out/q2
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/q2/pytest.log 2>&1; echo "exit $?" >> gpurun_out/q2/pytest.log
timeout 200 python scripts/time_apply.py c2 200 > gpurun_out/q2/ta.txt 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/q2/c2.json 2> gpurun_out/q2/c2.err
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q2/c3.json 2> gpurun_out/q2/c3.err
