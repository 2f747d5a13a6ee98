#!/bin/bash
# A/B the view-stream priority policies (NGS_STREAM_POLICY, experiments only) on c2.
for rep in 1 2; do
for p in ${POLICIES:-0 1 2 3}; do
  NGS_STREAM_POLICY=$p python tools/step_profile.py ${1:-c2} 5 2>&1 | grep "concurrent steps" | sed "s/^/policy $p: /"
done
done
