cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02w6
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "wave or early or smoother_paths" > gpurun_out/r02w6/pytest.log 2>&1
timeout 300 python scripts/wave_timeline.py c3 V > gpurun_out/r02w6/tl_c3_V.log 2>&1
timeout 300 python scripts/wave_timeline.py c3 D > gpurun_out/r02w6/tl_c3_D.log 2>&1
timeout 300 python scripts/time_wave.py c3 20 > gpurun_out/r02w6/time_c3.log 2>&1
tail -2 gpurun_out/r02w6/pytest.log; tail -3 gpurun_out/r02w6/tl_*.log; cat gpurun_out/r02w6/time_c3.log
