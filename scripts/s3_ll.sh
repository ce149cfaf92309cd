mkdir -p gpurun_out/ll
for k in 0 1; do
  if [ $k = 0 ]; then unset SDG_GS_MERGE; else export SDG_GS_MERGE=$k; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 300 --csv --log-file gpurun_out/ll/launch_k$k.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ll/ncu_k$k.log 2>&1
done
