#!/bin/bash
# dev: GS plan variants on the c2 apply
for b in 1 2 4; do
  echo "== bands=$b"
  SDG_GS_BANDS=$b timeout 120 python scripts/prof_apply.py c2 2>&1 | grep -E "^gs "
done
