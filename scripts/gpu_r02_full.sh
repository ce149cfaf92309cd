# full driver-style runs: our arm (with cpu_baseline) then the reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02f
( time timeout 1700 python bench.py --steps 20 --warmup 5 ) > gpurun_out/r02f/bench.json 2> gpurun_out/r02f/bench.err
echo "ours rc=$?"
( time timeout 1700 python bench.py --impl reference --steps 3 --warmup 1 ) > gpurun_out/r02f/ref.json 2> gpurun_out/r02f/ref.err
echo "ref rc=$?"
tail -3 gpurun_out/r02f/*.err
