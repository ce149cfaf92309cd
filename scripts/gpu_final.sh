#!/bin/bash
# end-of-session measurement: the round script, then configs 4 and 5s
bash scripts/gpu_round.sh
mkdir -p gpurun_out/c45
timeout 900 python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/c45/bench_c4.json 2> gpurun_out/c45/bench_c4.err
timeout 1500 python bench.py --config c5s --steps 1 --warmup 0 --no-cpu-baseline --coupling-iterations 200 > gpurun_out/c45/bench_c5s.json 2> gpurun_out/c45/bench_c5s.err
