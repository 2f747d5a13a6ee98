#!/bin/bash
# A/B timing helper (experiments only), run from the repo root on the GPU box:
#   tools/ab.sh "<bench args>" libA libB ...   (paper_2501_13975_b200/lib/libA.so, ... copied over the product lib in turn)
args="$1"; shift
L=paper_2501_13975_b200/lib
cp $L/libngs_b200.so /tmp/orig.so
for r in 1 2; do for v in "$@"; do
  cp $L/$v.so $L/libngs_b200.so
  python bench.py $args --no-cpu-baseline --no-solve-microbench 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done
cp /tmp/orig.so $L/libngs_b200.so
