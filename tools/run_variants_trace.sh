#!/bin/bash
# usage (on the GPU box): bash tools/run_variants_trace.sh default v1 v2 ... [-- extra prof_trace args]
args=()
vs=()
while [ $# -gt 0 ]; do if [ "$1" = "--" ]; then shift; args=("$@"); break; fi; vs+=("$1"); shift; done
for v in "${vs[@]}"; do
  if [ "$v" = default ]; then unset RT_B200_LIB; else export RT_B200_LIB=variants/$v/librt_b200.so; fi
  timeout 300 python tools/prof_trace.py "${args[@]}" 2>&1 | tail -1
done
