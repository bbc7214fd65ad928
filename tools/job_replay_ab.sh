#!/bin/bash
# Heavy-queue replay A/B on one box: frames of the same scene replay the last complete probe's
# queue (default) vs probing every frame (variants/noreplay); probe tests first.
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_probe.py tests/test_gpu_readback.py -x -q 2>&1 | tail -1
for r in 1 2; do
  for lib in "" variants/noreplay/librt_b200.so; do
    echo "== ${lib:-default}"; RT_B200_LIB=$lib timeout 300 python tools/eye_probe.py --soup --reps 17 2>&1 | tail -1
    RT_B200_LIB=$lib timeout 600 python bench.py --no-cpu --no-pt --no-e2e --steps 400 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2', round(d['value'],1), round(d['ms_per_step'],4), round(d['trace_mrays_s'],1))"
  done
done
