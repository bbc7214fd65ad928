#!/bin/bash
# Same-box A/B of the default bench step (config 2) across variant libraries:
#   bash tools/job_step_ab.sh TAG v1 v2 ...   (each run twice, interleaved)
cd "$(dirname "$0")/.."
tag=$1; shift
mkdir -p gpurun_out
for rep in 1 2; do for v in "$@"; do
  if [ $v = default ]; then unset RT_B200_LIB; else export RT_B200_LIB=variants/$v/librt_b200.so; fi
  echo "$v $(timeout 600 python bench.py --no-cpu --no-pt --no-e2e --steps 300 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"],4), round(d["lbvh_build_ms"],4), round(d["trace_mrays_s"],1))')"
done; done > gpurun_out/${tag}_step.log 2>&1
