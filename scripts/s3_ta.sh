mkdir -p gpurun_out/ta8
SDG_DEBUG=1 timeout 200 python scripts/time_apply.py c2 200 > gpurun_out/ta8/auto.txt 2>&1
for m in 1 4; do SDG_GS_MERGE=$m timeout 200 python scripts/time_apply.py c2 200 >> gpurun_out/ta8/out.txt 2>&1; done
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ta8/bench.json 2> gpurun_out/ta8/bench.err
