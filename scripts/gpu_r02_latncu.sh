cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02ln
timeout 600 ncu --kernel-name regex:k_gs_lattice --launch-skip 2 --launch-count 3 --set full --import-source on -f -o gpurun_out/r02ln/lat_c3 python scripts/one_apply.py c3 V 2 > gpurun_out/r02ln/ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02ln/v_c3.csv python scripts/one_apply.py c3 V 2 > /dev/null 2>&1
echo done
