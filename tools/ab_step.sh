#!/bin/bash
# A/B of library variants on tools/step_profile.py (concurrent + serialised stage times).
#   tools/ab_step.sh <config> libA libB ...
cfg=$1; shift
L=paper_2501_13975_b200/lib
cp $L/libngs_b200.so /tmp/orig.so
for r in 1 2; do for v in "$@"; do
  cp $L/$v.so $L/libngs_b200.so
  python tools/step_profile.py $cfg 5 2>&1 | grep -E "serialised|concurrent" | sed "s/^/$v: /" | cut -c1-400
done; done
cp /tmp/orig.so $L/libngs_b200.so
