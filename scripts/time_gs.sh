#!/bin/bash
# Dev: per-launch durations of the smoother kernels over one td_bgs apply (c2 by default).
cfg=${1:-c2}
SDG_PROFILER_RANGE=1 timeout 300 ncu --cache-control none --profile-from-start off --metrics gpu__time_duration.sum --csv \
  python scripts/prof_apply.py $cfg 2>/dev/null | grep -E "k_chain|k_gs_walk|k_gs_cluster" | \
  awk -F'","' '{n=$5; sub(/\(.*/,"",n); print n, $NF}' | sed 's/"//g'
