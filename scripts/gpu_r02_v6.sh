# full GPU suite, c4 per-apply profile, c5 (2000^2) first coupling iterations
cd $GRAFT_REPO_ROOT
O=gpurun_out/v6; mkdir -p $O
SDG_DEBUG=1 timeout 300 python scripts/time_apply.py c3 100 2>&1 | grep -E "label block|us/apply" | sed 's/^/c3 plan: /'
SDG_GS_PART_MERGE=0 timeout 300 python scripts/time_apply.py c3 100 2>&1 | grep -E "us/apply" | sed 's/^/c3 no part merge: /'
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
python -c "
import json; d=json.load(open('$O/bench_c3.json')); print('c3', d['ms_per_step'], d['details']['iterations'][:2], {k:(v['launches'],round(v['ms'],1)) for k,v in d['kernel_profile'].items() if k in ('gs','gs_wave','gs_lattice','coarse','gsprep')})"
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
SDG_DEBUG=1 timeout 900 python scripts/prof_apply.py c4 > $O/prof_c4.log 2>&1; echo "prof c4 rc=$?"
grep -E "launches/apply|label block|hier|gs wave|lattice\]" $O/prof_c4.log | head -40
timeout 1500 python bench.py --config c5 --steps 1 --warmup 0 --coupling-iterations 2 > $O/bench_c5_first2.json 2> $O/bench_c5_first2.err; echo "c5 rc=$?"
head -c 1200 $O/bench_c5_first2.json; tail -3 $O/bench_c5_first2.err
echo "--- c4s variants"
for s in -1 5 6; do
  A=""; [ $s -ge 0 ] && A="$s"
  timeout 300 python scripts/c4s_variants.py default $A 2>/dev/null | tail -1
  SDG_GS_EXACT=1 timeout 600 python scripts/c4s_variants.py gs_exact $A 2>/dev/null | tail -1
  SDG_TD_SPLIT=0 timeout 300 python scripts/c4s_variants.py no_split $A 2>/dev/null | tail -1
  SDG_GS_EXACT=1 SDG_TD_SPLIT=0 timeout 600 python scripts/c4s_variants.py gs_exact_no_split $A 2>/dev/null | tail -1
done
