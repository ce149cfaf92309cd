#!/bin/bash
# One GPU session: tests, smoke, bench (both arms), launch list, ncu captures.
# Output under gpurun_out/r (dev driver script; summaries are copied to profiles/).
set -x
mkdir -p gpurun_out/r
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r/smoke.log
timeout 600 python bench.py > gpurun_out/r/bench.json 2> gpurun_out/r/bench.err; echo "bench exit $?" >> gpurun_out/r/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r/bench_ref.json 2> gpurun_out/r/bench_ref.err
# launch list of one solve (after setup + the warm-up solve)
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r/plain_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 9000 -c 1200 --csv --log-file gpurun_out/r/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gs_walk -s 16 -c 4 -o gpurun_out/r/gs_full \
    python scripts/prof_apply.py c2 > gpurun_out/r/ncu_gs.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 20 -c 2 -o gpurun_out/r/spmv_full \
    python scripts/prof_apply.py c2 > gpurun_out/r/ncu_spmv.log 2>&1
ls -la gpurun_out/r
