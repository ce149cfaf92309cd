#!/bin/bash
# walk shape sweep for the velocity levels of c2 (time of a td_bgs apply)
mkdir -p gpurun_out/shape
for sh in "" "3,1,1,51520" "4,1,1,51520" "6,1,1,51520" "8,1,1,51520" "3,2,1,51520" "2,2,2,51520" "1,1,1,8852" "1,2,2,8852" "3,1,1,8852" "1,1,2,8852" "2,2,1,8852"; do
  echo "== $sh" >> gpurun_out/shape/out.txt
  SDG_WALK_SHAPE=$sh timeout 200 python scripts/time_apply.py c2 200 2>&1 | grep us/apply >> gpurun_out/shape/out.txt
done
