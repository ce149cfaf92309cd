cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02l
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02l/v_c3.csv python scripts/one_apply.py c3 V 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02l/d_c3.csv python scripts/one_apply.py c3 D 2 > /dev/null 2>&1
echo done
