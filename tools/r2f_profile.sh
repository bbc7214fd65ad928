#!/bin/bash
# Session-3 ncu re-captures of the eye megakernel (config 2 sphere, config 4 soup) after the
# heavy-queue replay / probe-skip hint / PDL frame launch, plus the launch list of two bench
# steps.  GPU box, one GPU, --clock-control none.  Outputs under gpurun_out/.
set -x
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:pt_megakernel --launch-skip 2 --launch-count 1 \
    -o gpurun_out/r2f_mega_eye -f python tools/drive_render.py eye 3 > gpurun_out/r2f_ncu_eye.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pt_megakernel --launch-skip 2 --launch-count 1 \
    -o gpurun_out/r2f_soup_trace -f python tools/drive_render.py soup 3 > gpurun_out/r2f_ncu_soup.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2f_launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-pt --no-e2e > gpurun_out/r2f_ncu_launch_bench.log 2>&1
