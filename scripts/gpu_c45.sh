#!/bin/bash
# configs 4 and 5s, one measured run each (minutes of GPU time apiece)
mkdir -p gpurun_out/c45
timeout 900 python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/c45/bench_c4.json 2> gpurun_out/c45/bench_c4.err
timeout 1200 python bench.py --config c5s --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/c45/bench_c5s.json 2> gpurun_out/c45/bench_c5s.err
