#!/bin/bash
# Same-box A/B of trace/render timings across variant libraries (tools/variants.sh):
#   bash tools/ab_trace.sh OUT "--soup" default v1 v2 ...   (each variant run twice, interleaved)
out=$1; flags=$2; shift 2
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
  for v in "$@"; do
    if [ $v = default ]; then unset RT_B200_LIB; else export RT_B200_LIB=variants/$v/librt_b200.so; fi
    timeout 300 python tools/prof_trace.py $flags --reps 11
  done
done > gpurun_out/$out 2>&1
