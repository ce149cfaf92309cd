mkdir -p gpurun_out/q
SDG_DEBUG=1 timeout 200 python scripts/time_apply.py c2 200 > gpurun_out/q/ta.txt 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q/c2.json 2> gpurun_out/q/c2.err
SDG_DEBUG=1 timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q/c3.json 2> gpurun_out/q/c3.err
