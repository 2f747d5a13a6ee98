#!/bin/bash
# c5 stage timings for several library builds (experiments only): tools/ab_c5.sh libA libB ...
L=paper_2501_13975_b200/lib
cp $L/libngs_b200.so /tmp/orig_c5.so
for v in "$@"; do cp $L/$v.so $L/libngs_b200.so; echo "$v"; python tools/c5_bench.py 3 | tail -2; done
cp /tmp/orig_c5.so $L/libngs_b200.so
