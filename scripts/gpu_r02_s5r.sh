cd $GRAFT_REPO_ROOT
O=gpurun_out/s5r; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "early or apply or determinism" 2>&1 | tail -1
for k in 1 2 3; do SDG_DEBUG=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2> $O/err$k.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c3', round(d['ms_per_step'],2), d['details']['iterations'][:1])"; grep "interface correction" $O/err$k.log; done
SDG_DEBUG=1 timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2> $O/errc2.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c2', round(d['ms_per_step'],2), d['details']['iterations'][:1])"; grep "interface correction" $O/errc2.log
