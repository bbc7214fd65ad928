#!/bin/bash
# Tile-probe A/B on one GPU box: eye frames (1080p sphere, 4K soup) with the probe off / on
# (RT_PROBE_BUDGET env), frame hashes must agree; then the default bench step both ways.
#   bash tools/job_probe_ab.sh TAG
cd "$(dirname "$0")/.."
tag=${1:-probe}
mkdir -p gpurun_out
for b in 0 24 0 24; do RT_PROBE_BUDGET=$b timeout 300 python tools/eye_probe.py --soup --reps 11; done \
    > gpurun_out/${tag}_frames.log 2>&1
for b in 0 24; do
  RT_PROBE_BUDGET=$b timeout 300 python bench.py --no-cpu --no-pt --no-e2e --steps 300 2>/dev/null
done > gpurun_out/${tag}_bench.log 2>&1
