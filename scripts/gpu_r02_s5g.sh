cd $GRAFT_REPO_ROOT
for w in 1 2 4; do
echo "SDG_WAVE_W=$w"; SDG_WAVE_W=$w timeout 120 python scripts/time_wave.py c3 2>&1 | grep default
done
for w in 1 2; do
SDG_WAVE_W=$w timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c3 W=$w', d['ms_per_step'], d['details']['iterations'][:2], d['kernel_profile']['gs_wave'])"
done
