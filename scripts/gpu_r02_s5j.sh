# session 5: MAC block size / ring depth variants (separate builds of gs_wave.cu)
cd $GRAFT_REPO_ROOT
P=paper_2108_13229_b200
cp $P/libsdgpu.so /tmp/libsdgpu_base.so
for v in base ku16d4; do
  if [ $v = base ]; then cp /tmp/libsdgpu_base.so $P/libsdgpu.so; else cp $P/libsdgpu_$v.so $P/libsdgpu.so; fi
  echo "== $v"
  timeout 120 python scripts/time_wave.py c3 2>&1 | grep "V.*default"
  timeout 200 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "wave" 2>&1 | tail -1
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c3 $v', d['ms_per_step'], d['details']['iterations'][:2], d['kernel_profile']['gs_wave'])"
done
cp /tmp/libsdgpu_base.so $P/libsdgpu.so
