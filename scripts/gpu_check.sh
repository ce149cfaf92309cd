#!/bin/bash
# full GPU check of the current tree: tests, smoke, default bench
mkdir -p gpurun_out/chk
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/chk/pytest.log 2>&1; echo "exit $?" >> gpurun_out/chk/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk/smoke.log 2>&1; echo "exit $?" >> gpurun_out/chk/smoke.log
timeout 600 python bench.py > gpurun_out/chk/bench.json 2> gpurun_out/chk/bench.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/chk/bench_c3.json 2> gpurun_out/chk/bench_c3.err
