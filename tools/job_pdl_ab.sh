#!/bin/bash
# Render-launch A/B on one box: counters zeroed by a PDL kernel + PDL frame launch (default)
# vs the same without programmatic serialization (variants/nopdl); config-2 bench value.
cd "$(dirname "$0")/.."
for r in 1 2; do
  for v in default nopdl; do
    if [ $v = default ]; then lib=""; else lib="RT_B200_LIB=variants/nopdl/librt_b200.so"; fi
    echo "== $v"; env $lib timeout 300 python bench.py --no-cpu --no-pt --no-e2e --steps 400 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],4), round(d['lbvh_build_ms'],4), round(d['trace_mrays_s'],1))"
  done
done
