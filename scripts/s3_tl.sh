mkdir -p gpurun_out/tl
for sp in 0 1; do SDG_TD_SPLIT=$sp timeout 200 python scripts/walk_timeline.py > gpurun_out/tl/split$sp.txt 2>&1; done
for sp in 0 1; do SDG_TD_SPLIT=$sp timeout 200 python scripts/time_apply.py c2 200 >> gpurun_out/tl/ta.txt 2>&1; done
