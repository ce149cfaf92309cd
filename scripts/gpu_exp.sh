#!/bin/bash
# dev: c2 bench + apply launch durations + c4 (one run) for an experiment build
mkdir -p gpurun_out/e
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/e/bench.json 2> gpurun_out/e/bench.err
SDG_PROFILER_RANGE=1 timeout 600 ncu --profile-from-start off --clock-control none --csv --log-file gpurun_out/e/apply_dram.csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum python scripts/prof_apply.py c2 > gpurun_out/e/ncu_apply.log 2>&1
if [ "$1" = "c4" ]; then
timeout 1200 python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/e/bench_c4.json 2> gpurun_out/e/bench_c4.err
fi
