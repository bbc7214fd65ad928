#!/bin/bash
# Re-probe interval A/B (config-2 bench): every 8th frame (default) vs 16 / 32 (variants)
cd "$(dirname "$0")/.."
for r in 1 2; do
  for lib in "" variants/rp16/librt_b200.so variants/rp32/librt_b200.so; do
    echo -n "${lib:-default}: "; RT_B200_LIB=$lib timeout 300 python bench.py --no-cpu --no-pt --no-e2e --steps 800 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],4))"
  done
done
