#!/bin/bash
# Probe-budget sweep under heavy-queue replay (config-2 bench value; env RT_PROBE_BUDGET)
cd "$(dirname "$0")/.."
for r in 1 2; do
  for b in 12 16 24 32 48; do
    echo -n "budget $b: "; RT_PROBE_BUDGET=$b timeout 300 python bench.py --no-cpu --no-pt --no-e2e --steps 400 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],4), round(d['trace_mrays_s'],1))"
  done
done
