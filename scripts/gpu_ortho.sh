#!/bin/bash
mkdir -p gpurun_out/orth
timeout 900 python -m pytest tests -m gpu -q -x -k "gmres or c3 or dist or transient" > gpurun_out/orth/pytest.log 2>&1; echo "exit $?" >> gpurun_out/orth/pytest.log
timeout 600 python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/orth/c3.json 2> gpurun_out/orth/c3.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_multi" -s 200 -c 40 --csv --log-file gpurun_out/orth/ortho.csv python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/orth/ncu.log 2>&1
