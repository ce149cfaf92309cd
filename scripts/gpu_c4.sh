#!/bin/bash
mkdir -p gpurun_out/c4s
timeout 900 python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/c4s/bench_c4.json 2> gpurun_out/c4s/bench_c4.err
timeout 200 python scripts/time_apply.py c2 200 > gpurun_out/c4s/ta.txt 2>&1
