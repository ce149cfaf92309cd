mkdir -p gpurun_out/dyn
for cfg in "4 0" "4 6" "4 8" "8 6" "8 8" "16 8"; do set -- $cfg
  SDG_DEBUG=1 SDG_GS_MERGE=$1 SDG_GS_MERGE_CAP=$2 timeout 200 python scripts/time_apply.py c2 200 > gpurun_out/dyn/k$1_c$2.txt 2>&1
done
SDG_GS_MERGE=8 SDG_GS_MERGE_CAP=8 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 60 --csv --log-file gpurun_out/dyn/launch_k8c8.csv python scripts/time_apply.py c2 20 > gpurun_out/dyn/ncu.log 2>&1
