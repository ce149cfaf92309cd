mkdir -p gpurun_out/sell3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_sell -s 30 -c 1 -o gpurun_out/sell3/spmv_c3 python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/sell3/ncu.log 2>&1
