# session 5: early interface correction on/off at c3, c2, c4s-like sizes
cd $GRAFT_REPO_ROOT
run() { cfgname=$1; shift; env "$@" timeout 600 python bench.py --config $cfgname --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); kp=d['kernel_profile']; print('$cfgname $*', round(d['ms_per_step'],2), d['details']['iterations'][:1], {k:round(kp[k]['ms'],1) for k in ('gs','gs_wave','coarse','iface') if k in kp})"; }
run c3 SDG_NOP=1
run c3 SDG_TD_EARLY=0
run c3 SDG_NOP=1
run c3 SDG_TD_EARLY=0
run c2 SDG_NOP=1
run c2 SDG_TD_EARLY=0
