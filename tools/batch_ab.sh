#!/bin/bash
# A/B: batched secondary backward (NGS_BATCH_SECONDARIES) x stream priority policy (NGS_STREAM_POLICY)
for r in 1 2; do for c in 0 1; do for p in 0 1 2 3; do
  NGS_STREAM_POLICY=$p NGS_BATCH_SECONDARIES=$c python tools/step_profile.py ${1:-c2} 5 2>&1 | grep -E "concurrent steps" | sed "s/^/batch $c policy $p: /" | cut -c1-260
done; done; done
