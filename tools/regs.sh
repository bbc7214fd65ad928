#!/bin/bash
# ptxas register/spill summary per kernel: tools/regs.sh csrc/render.cu
f=$1
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -Xptxas -v -c "$f" -o /tmp/regs_$$.o 2>&1 |
  awk '/Compiling entry function/ {match($0, /_Z[^'"'"']*/); name=substr($0, RSTART, 60)} /Used [0-9]+ registers/ {match($0, /Used [0-9]+ registers/); r=substr($0, RSTART, RLENGTH)} /spill stores/ {match($0, /[0-9]+ bytes spill stores/); sp=substr($0, RSTART, RLENGTH); print name, "|", r, "|", sp}' | sort -u
rm -f /tmp/regs_$$.o
