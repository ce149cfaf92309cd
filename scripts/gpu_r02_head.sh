set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02
lscpu > gpurun_out/r02/lscpu.txt; nproc >> gpurun_out/r02/lscpu.txt
nvidia-smi > gpurun_out/r02/smi.txt
(timeout 1500 taskset -c 2 python scripts/ref_c3_probe.py > gpurun_out/r02/ref_c3_probe.log 2>&1 &)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02/pytest_head.log 2>&1
timeout 400 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02/bench_c3_head.json 2> gpurun_out/r02/bench_c3_head.err
while pgrep -f ref_c3_probe > /dev/null; do sleep 10; done
cat gpurun_out/r02/ref_c3_probe.log
