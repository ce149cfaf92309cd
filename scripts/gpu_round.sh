#!/bin/bash
# One GPU session: tests, smoke, bench (both arms, c2 and c3), launch list, ncu captures.
# Output under gpurun_out/r (dev driver script; summaries are copied to profiles/).
set -x
mkdir -p gpurun_out/r
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r/smoke.log
timeout 600 python bench.py > gpurun_out/r/bench.json 2> gpurun_out/r/bench.err; echo "bench exit $?" >> gpurun_out/r/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r/bench_ref.json 2> gpurun_out/r/bench_ref.err
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/r/bench_c3.json 2> gpurun_out/r/bench_c3.err
# launch list of one solve (after setup + the warm-up solve)
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r/plain_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 9000 -c 1200 --csv --log-file gpurun_out/r/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r/ncu_launches.log 2>&1
# DRAM bytes + duration of every kernel of one preconditioner apply
SDG_PROFILER_RANGE=1 timeout 600 ncu --profile-from-start off --clock-control none --csv --log-file gpurun_out/r/apply_dram.csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum python scripts/prof_apply.py c2 > gpurun_out/r/ncu_apply.log 2>&1
# full capture of the velocity pre-smoother walk (5th walk of an apply: the D cycle is issued first, on the side stream)
SDG_PROFILER_RANGE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:k_gs_walk -s 4 -c 1 -o gpurun_out/r/gs_walk_v0 python scripts/prof_apply.py c2 > gpurun_out/r/ncu_gs.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_sell -s 30 -c 1 -o gpurun_out/r/spmv_c3 \
    python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r/ncu_spmv.log 2>&1
# the interface GEMV at c3 (K = 250,000 x 500 fp64 = 1 GB, streamed once per apply)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_colmajor_gemv_sub -s 20 -c 1 -o gpurun_out/r/gemv_c3 \
    python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r/ncu_gemv.log 2>&1
timeout 1200 python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r/bench_c4.json 2> gpurun_out/r/bench_c4.err
ls -la gpurun_out/r
