#!/bin/bash
# Registers / spills per kernel of one CUDA source (sm_100a): tools/regs.sh file.cu [filter]
f=$1; flt=${2:-.}
nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -fPIC -Xptxas -v -I "$(dirname "$0")/../include" -c "$f" -o /tmp/regs_$$.o 2>&1 |
  awk '/Compiling entry function/ {match($0, /_Z[^'"'"']*/); name=substr($0, RSTART, RLENGTH)}
       /spill stores/ {sp=$0; sub(/.*frame, /, "", sp)}
       /Used [0-9]+ registers/ {match($0, /Used [0-9]+ registers/); print substr($0, RSTART+5, RLENGTH-15) "\t" sp "\t" name}' |
  c++filt | grep -E "$flt" | sed 's/(anonymous namespace):://g' | cut -c1-160
rm -f /tmp/regs_$$.o
