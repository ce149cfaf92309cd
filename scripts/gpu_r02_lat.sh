cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02lat
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/r02lat/pytest.log 2>&1
echo "pytest rc=$?"
SDG_DEBUG=1 timeout 300 python scripts/time_wave.py c3 20 > gpurun_out/r02lat/time_c3.log 2> gpurun_out/r02lat/time_c3.err
timeout 300 python scripts/time_wave.py c2 50 > gpurun_out/r02lat/time_c2.log 2>&1
timeout 300 python scripts/wave_timeline.py c3 V > gpurun_out/r02lat/tl_c3_V.log 2>&1
tail -3 gpurun_out/r02lat/pytest.log; cat gpurun_out/r02lat/time_c3.log gpurun_out/r02lat/time_c2.log; head -4 gpurun_out/r02lat/tl_c3_V.log
