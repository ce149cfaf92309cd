# session 5: nested-dissection leaf size (SDG_ND_LEAF) at c3 and c4
cd $GRAFT_REPO_ROOT
run() { env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); kp=d['kernel_profile']; print('c3 $*', round(d['ms_per_step'],2), d['details']['iterations'][:1], {k:round(kp[k]['ms'],1) for k in ('coarse',) if k in kp}, d['details'].get('setup_s'))"; }
run SDG_ND_LEAF=1024
run SDG_ND_LEAF=2048
run SDG_ND_LEAF=1024
run SDG_ND_LEAF=2048
run SDG_ND_LEAF=1536
for l in 1024 2048; do SDG_ND_LEAF=$l timeout 400 python scripts/time_apply.py c4 60 2>&1 | grep "us/apply" | sed "s/^/c4 leaf $l: /"; done
for l in 1024 2048; do SDG_ND_LEAF=$l timeout 300 python scripts/time_apply.py c2 200 2>&1 | grep "us/apply" | sed "s/^/c2 leaf $l: /"; done
