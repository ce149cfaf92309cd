#!/bin/bash
mkdir -p gpurun_out/c5
timeout 1500 python bench.py --config c5s --steps 1 --warmup 0 --no-cpu-baseline --coupling-iterations 200 > gpurun_out/c5/bench_c5s.json 2> gpurun_out/c5/bench_c5s.err
