#!/bin/bash
# quick iteration: GPU tests, apply timing, c2/c3 bench (no CPU baseline)
mkdir -p gpurun_out/q
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/q/pytest.log 2>&1; echo "exit $?" >> gpurun_out/q/pytest.log
timeout 200 python scripts/time_apply.py c2 200 > gpurun_out/q/ta.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/q/c2.json 2> gpurun_out/q/c2.err
timeout 600 python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/q/c3.json 2> gpurun_out/q/c3.err
