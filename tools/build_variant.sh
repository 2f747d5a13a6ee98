#!/bin/bash
# Build libngs_b200.so with extra nvcc flags into paper_2501_13975_b200/lib/<name>.so (A/B experiments).
#   tools/build_variant.sh <name> [-DFOO=1 ...]
name=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
C=$R/paper_2501_13975_b200/csrc
T=$(mktemp -d)
for f in render sort loss backward solve context; do
  nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -Xcompiler -O3 "$@" \
    -I $R/include -c $C/$f.cu -o $T/$f.o || exit 1
done
nvcc -shared -gencode arch=compute_100a,code=sm_100a $T/*.o -o $R/paper_2501_13975_b200/lib/$name.so
rm -rf $T
