#!/bin/bash
# ncu captures for profiles/ (GPU box, one GPU): one config-2 build and one config-4 build
# (--set full, cold caches, the second build of each process), and the launch list of two
# bench.py config-2 steps (gpu__time_duration only).  Outputs under gpurun_out/.
set -x
K='regex:lbvh_|onesweep'
ncu --set full --clock-control none --import-source on -k "$K" --launch-skip 8 --launch-count 8 \
    -o gpurun_out/r1_build -f python tools/drive_build.py 2 30 > gpurun_out/ncu_build.log 2>&1
ncu --set full --clock-control none --import-source on -k "$K" --launch-skip 8 --launch-count 8 \
    -o gpurun_out/r1_soup_build -f python tools/drive_build.py 2 30 soup > gpurun_out/ncu_soup_build.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-pt --no-e2e > gpurun_out/ncu_launch_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pt_megakernel --launch-skip 1 --launch-count 1 \
    -o gpurun_out/r1_mega_eye -f python tools/drive_render.py eye 2 > gpurun_out/ncu_eye.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pt_megakernel --launch-skip 1 --launch-count 1 \
    -o gpurun_out/r1_mega_pt -f python tools/drive_render.py pt 2 > gpurun_out/ncu_pt.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pt_megakernel --launch-skip 1 --launch-count 1 \
    -o gpurun_out/r1_soup_trace -f python tools/drive_render.py soup 2 > gpurun_out/ncu_soup.log 2>&1
