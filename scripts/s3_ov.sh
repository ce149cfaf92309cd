mkdir -p gpurun_out/ov
for ov in 0 1; do for gr in 0 1; do
  SDG_TD_OVERLAP=$ov SDG_GRAPHS=$gr timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ov/ov${ov}_g${gr}.json 2> gpurun_out/ov/ov${ov}_g${gr}.err
done; done
