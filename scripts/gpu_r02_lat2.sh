cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02lat2
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py tests/test_gpu_transient.py -q -k "lattice or ilu0 or rhs or bicgstab_matches or gmres50" > gpurun_out/r02lat2/pytest.log 2>&1
echo "pytest rc=$?"
timeout 300 python scripts/time_wave.py c3 20 > gpurun_out/r02lat2/time_c3.log 2>&1
timeout 300 python scripts/time_wave.py c2 50 > gpurun_out/r02lat2/time_c2.log 2>&1
SDG_GS_LATTICE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02lat2/v_c3.csv python scripts/one_apply.py c3 V 2 > /dev/null 2>&1
tail -5 gpurun_out/r02lat2/pytest.log; cat gpurun_out/r02lat2/time_c3.log gpurun_out/r02lat2/time_c2.log
