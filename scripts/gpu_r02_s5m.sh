cd $GRAFT_REPO_ROOT
O=gpurun_out/s5m; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
SDG_DEBUG=1 timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"; grep "interface correction" $O/bench_c3.err
SDG_DEBUG=1 timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err; echo "c2 rc=$?"; grep "interface correction" $O/bench_c2.err
SDG_DEBUG=1 timeout 600 python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc=$?"; grep "interface correction" $O/bench_c4.err
for f in bench_c3 bench_c2 bench_c4; do python -c "
import json; d=json.loads(open('$O/$f.json').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['e2e'] and d['e2e'].get('ms_per_step'))"; done
timeout 300 python scripts/e2e_probe.py c3 | tail -4
