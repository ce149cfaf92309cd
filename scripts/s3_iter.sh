# quick iteration: bench (auto), overlap off, launch list, GPU tests
mkdir -p gpurun_out/it
SDG_DEBUG=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/it/auto.json 2> gpurun_out/it/auto.err
SDG_TD_OVERLAP=0 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/it/noov.json 2> gpurun_out/it/noov.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 200 --csv --log-file gpurun_out/it/launch.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/it/ncu.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_solvers.py::test_c3_full_size_matches_reference_fingerprint > gpurun_out/it/pytest.log 2>&1; echo "exit $?" >> gpurun_out/it/pytest.log
