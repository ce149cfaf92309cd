# driver-style runs at the driver's flags: our arm (with cpu_baseline), then the reference arm
cd $GRAFT_REPO_ROOT
O=gpurun_out/full; mkdir -p $O
( time timeout 1750 python bench.py --gpus 1 --steps 20 --warmup 5 ) > $O/bench.json 2> $O/bench.err; echo "ours rc=$?"
( time timeout 1750 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > $O/ref.json 2> $O/ref.err; echo "ref rc=$?"
tail -4 $O/bench.err $O/ref.err
head -c 300 $O/bench.json; echo; head -c 600 $O/ref.json
